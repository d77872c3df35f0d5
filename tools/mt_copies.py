"""32 copies of one shot: in a deviating run, which copies deviate (per shot? per warp of 8?)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np

from paper_1406_6923_b200 import CoupledStepper, SourceTerm, project_source
from paper_1406_6923_b200.configs import locate, make_workload
from paper_1406_6923_b200.pulses import ricker
from test_fullsize_gpu import _build

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 60
wl3, models, dt, _, probes = _build(3, extra_sources=make_workload(4).sources)
wl = make_workload(4)
a, r = locate(wl.sources[0], wl.counts, wl.p)
sh = SourceTerm(a, project_source(models[a], r), ricker(wl.f0, wl.delay))
with CoupledStepper(models, dt) as st:
    for i in range(rep):
        _, rows, norms = st.run_shots(n, [sh] * 32, probes=probes, return_norms=True)
        ref = np.median(rows, axis=1, keepdims=True)  # the value most copies agree on
        dev = rows != ref
        if not dev.any():
            continue
        k, q, p = np.nonzero(dev)
        k0 = k.min()
        print(f"run {i}: deviating copies overall {sorted(set(q.tolist()))}; first at record {k0}: copies {sorted(set(q[k == k0].tolist()))} "
              f"probes {len(set(p[k == k0].tolist()))}; norms deviating copies "
              f"{sorted(set(np.nonzero(norms != np.median(norms, axis=1, keepdims=True))[1].tolist()))}")
