"""Time the explicit-operator transfer maps (ntd_full_band) on a config-1 subdomain (N = 4913).

    python tools/ntd_bench.py      (on a B200; prints one JSON line)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_1406_6923_b200 import grid as pg  # noqa: E402
from paper_1406_6923_b200.configs import make_workload  # noqa: E402
from paper_1406_6923_b200.ntd import ntd_full_band  # noqa: E402

wl = make_workload(1)
ext = tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing))
part = pg.build_partition(pg.DomainSpec(ext, wl.counts, wl.p))
op = pg.assemble_subdomain_operator(part, (0, 0, 0), wl.c_field, with_matrix=True)
rng = np.random.default_rng(0)
f = rng.standard_normal((op.n_nodes, 6 * wl.modes_per_face))
out = {"n": op.n_nodes, "w": f.shape[1]}
ntd_full_band(op.matrix, f, [30.0])  # warm-up (module load)
for k in (1, 20, 148):
    om = np.geomspace(20.0, 400.0, k)
    t0 = time.perf_counter()
    ntd_full_band(op.matrix, f, om)
    out[f"{k}_omegas_s"] = time.perf_counter() - t0
print(json.dumps(out))
