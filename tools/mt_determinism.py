"""Run-to-run determinism probe for the multi-shot kernel (config 4 at full size).

    python tools/mt_determinism.py [n_steps] [repeats]
Runs run_shots several times on one stepper and reports where the probe rows differ.
"""
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
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 6
wl3, models, dt, _, probes = _build(3, extra_sources=make_workload(4).sources)
wl = make_workload(4)
shots = []
for ijk in wl.sources:
    a, r = locate(ijk, wl.counts, wl.p)
    shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl.f0, wl.delay)))
with CoupledStepper(models, dt) as st:
    ref = None
    for i in range(rep):
        _, rows, norms = st.run_shots(n, shots, probes=probes, return_norms=True)
        print("run", i, "nan", int(np.isnan(rows).sum()), "ms/step", st.last_kernel_ms / n)
        if ref is None:
            ref, refn = rows.copy(), norms.copy()
            continue
        d = rows != ref
        if d.any():
            k, q, p = np.nonzero(d)
            print("  differing entries", int(d.sum()), "first step", k.min(), "shots", sorted(set(q.tolist()))[:40])
            i0 = np.argmin(k)
            print("  first:", k[i0], q[i0], p[i0], rows[k[i0], q[i0], p[i0]], ref[k[i0], q[i0], p[i0]],
                  "probe sub", probes[p[i0]].alpha)
            mk = k == k.min()
            print("  at first step: probes", sorted(set(p[mk].tolist()))[:20], "subs",
                  sorted(set(probes[j].alpha for j in p[mk]))[:20])
            rel = np.abs(rows - ref)[d] / np.maximum(np.abs(ref[d]), 1e-300)
            print("  rel diff max", rel.max(), "median", np.median(rel), "max abs diff / max |rows| per shot",
                  max(np.abs(rows[:, qq] - ref[:, qq]).max() / np.abs(ref[:, qq]).max() for qq in set(q.tolist())))
        dn = norms != refn
        if dn.any():
            k, q = np.nonzero(dn)
            print("  norms differ from step", k.min(), "shots at that step", sorted(set(q[k == k.min()].tolist())),
                  "max rel", (np.abs(norms - refn)[dn] / refn[dn]).max())
        else:
            print("  norms identical")
