"""Run-to-run repeatability of the multi-shot kernel at config-4 size: N runs of K steps on one
stepper, hashed (probe rows + per-shot norms); prints how many distinct results were seen.

    python tools/mt_stress.py [steps=30] [runs=300]
"""
import collections
import hashlib
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np

from paper_1406_6923_b200 import CoupledStepper, SourceTerm, project_source
from paper_1406_6923_b200.configs import locate, make_workload
from paper_1406_6923_b200.pulses import ricker
from test_fullsize_gpu import _build
import paper_1406_6923_b200.stepper as _ps
if os.environ.get('MT_NOLIMIT'):
    _ps.GROWTH_LIMIT = float('inf')

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rep = int(sys.argv[2]) if len(sys.argv) > 2 else 300
wl3, models, dt, _, probes = _build(3, extra_sources=make_workload(4).sources)
wl = make_workload(4)
shots = []
for ijk in wl.sources:
    a, r = locate(ijk, wl.counts, wl.p)
    shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl.f0, wl.delay)))
with CoupledStepper(models, dt) as st:
    hs = collections.Counter()
    nans = 0
    ms = []
    for i in range(rep):
        _, rows, norms = st.run_shots(n, shots, probes=probes, return_norms=True)
        ms.append(st.last_kernel_ms / n)
        nans += int(np.isnan(rows).sum() + np.isnan(norms).sum())
        hs[hashlib.md5(rows.tobytes() + norms.tobytes()).hexdigest()[:8]] += 1
    print(f"{rep} runs of {n} steps: distinct results {len(hs)}, counts {sorted(hs.values(), reverse=True)[:8]}, "
          f"ms/step {np.median(ms):.4f}, NaNs {nans}")
