"""Run-to-run repeatability of the batched GPU ROM build (DMMA GEMMs, DMMA PCG line passes, CholQR2):
N builds of the first M subdomains of a config, hashed (Gamma, Gamma-hat, G, A_j, B_j).

    python tools/rom_stress.py [cfg=3] [subdomains=512] [runs=20]
"""
import collections
import hashlib
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1406_6923_b200 import build_models  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m = int(sys.argv[2]) if len(sys.argv) > 2 else 512
rep = int(sys.argv[3]) if len(sys.argv) > 3 else 20
wl, ops, alphas, _, _ = bench._workload(cfg)
hs = collections.Counter()
first = None
worst = 0.0
for i in range(rep):
    models = build_models(ops[:m], wl.modes_per_face, wl.n, wl.shift)
    h = hashlib.md5()
    arrs = []
    for a in sorted(models):
        md = models[a]
        for x in (md.gammas, md.gamma_hats, md.scales, md.tdiag, md.toff):
            x = np.ascontiguousarray(x)
            h.update(x.tobytes())
            arrs.append(x)
    hs[h.hexdigest()[:8]] += 1
    if first is None:
        first = arrs
    else:
        worst = max(worst, max(float(np.abs(x - y).max() / max(np.abs(y).max(), 1e-300)) for x, y in zip(arrs, first)))
print(f"{rep} builds of {m} subdomains (config {cfg}): distinct results {len(hs)}, counts {sorted(hs.values(), reverse=True)[:8]}, "
      f"largest relative deviation from the first build {worst:.2e}")
