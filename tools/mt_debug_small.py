"""Multi-shot kernel against the single-source stepper on a small config-4-recipe domain.

    [SFW_STEP_MAXGRID=g] python tools/mt_debug_small.py nx ny nz [steps=60]
"""
import math
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np

import paper_1406_6923_b200.stepper as ps
from helpers import face_probes, rel
from paper_1406_6923_b200 import (CoupledStepper, Probe, SourceTerm, build_models, cfl_estimate_coupled,
                                  project_source)
from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200.configs import locate, make_workload
from paper_1406_6923_b200.pulses import ricker

counts = tuple(int(v) for v in sys.argv[1:4])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 60
ps.GROWTH_LIMIT = float("inf")
wl = make_workload(4, counts=counts)
ext = tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing))
part = pg.build_partition(pg.DomainSpec(ext, wl.counts, wl.p))
ops = [pg.assemble_subdomain_operator(part, a, wl.c_field) for a in sorted(s.alpha for s in part.subdomains)]
rows_req = {}
for ijk in wl.sources:
    a, r = locate(ijk, wl.counts, wl.p)
    rows_req.setdefault(a, []).append(r)
models = build_models(ops, 9, 8, wl.shift, rows=rows_req)
lam, _ = cfl_estimate_coupled(models)
dt = 0.9 * 2.0 / math.sqrt(lam)
shots = []
for ijk in wl.sources:
    a, r = locate(ijk, wl.counts, wl.p)
    shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl.f0, wl.delay)))
probes = [Probe(a, w) for a, w in face_probes(models, wl)]
with CoupledStepper(models, dt) as st:
    _, rows, norms = st.run_shots(n, shots, probes=probes, return_norms=True)
    states = {q: st.shot_state(q) for q in (0, 13, 31)}
for q in (0, 13, 31):
    with CoupledStepper(models, dt, sources=(shots[q],)) as st1:
        _, r1 = st1.run(n, probes=probes)
        u1 = st1.u_curr
    big = max(np.abs(v).max() for v in u1.values())
    bad = [(a, float(np.abs(states[q][0][a] - u1[a]).max() / big)) for a in sorted(u1)
           if np.abs(states[q][0][a] - u1[a]).max() > 1e-8 * big]
    print(f"shot {q}: rows vs single-source {rel(rows[:, q, :], r1):.2e}; state max {big:.2e}; deviating subdomains "
          f"{len(bad)}: {bad[:8]}")
