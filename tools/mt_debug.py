"""Locate deviations of the multi-shot kernel at config-4 size: shot q of run_shots against the
single-source stepper, per step (probe rows) and per subdomain / layer (final state).

    python tools/mt_debug.py [steps=4] [shot=0]
"""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np

import paper_1406_6923_b200.stepper as ps
from paper_1406_6923_b200 import CoupledStepper, SourceTerm, project_source
from paper_1406_6923_b200.configs import locate, make_workload
from paper_1406_6923_b200.pulses import ricker
from test_fullsize_gpu import _build

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
q = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ps.GROWTH_LIMIT = float("inf")
wl3, models, dt, _, probes = _build(3, extra_sources=make_workload(4).sources)
wl = make_workload(4)
shots = []
for ijk in wl.sources:
    a, r = locate(ijk, wl.counts, wl.p)
    shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl.f0, wl.delay)))
with CoupledStepper(models, dt) as st:
    _, rows, norms = st.run_shots(n, shots, probes=probes, return_norms=True)
    uq, upq = st.shot_state(q)
with CoupledStepper(models, dt, sources=(shots[q],)) as st1:
    _, r1 = st1.run(n, probes=probes)
    u1, up1 = st1.u_curr, st1.u_prev
jump = np.argwhere(norms[1:] > 50 * np.maximum(norms[:-1], 1e-300))
print("norm jumps (step, shot):", [(int(a) + 2, int(b), float(norms[a + 1, b])) for a, b in jump[:20]])
for qq in range(32):
    with np.errstate(all="ignore"):
        pass
for k in range(n + 1):
    d = np.abs(rows[k, q] - r1[k]).max()
    print(f"step {k}: max |row diff| {d:.3e}  max |row| {np.abs(r1[k]).max():.3e}  norm {norms[k - 1, q] if k else 0:.6e}")
w = 54
for name, ua, ub in (("u_curr", uq, u1), ("u_prev", upq, up1)):
    bad = []
    for a in sorted(ub):
        d = np.abs(ua[a] - ub[a])
        if d.max() > 1e-12 * max(1e-300, max(np.abs(v).max() for v in ub.values())):
            lay = sorted(set((np.nonzero(d > 0.5 * d.max())[0] // w).tolist()))
            bad.append((a, float(d.max()), lay, len(models[a].neighbors)))
    print(name, "deviating subdomains:", len(bad), "of", len(ub))
    for b in bad[:40]:
        print("   ", b)
print("source subdomain of the shot:", shots[q].alpha)
