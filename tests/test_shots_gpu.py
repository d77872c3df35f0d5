"""Multi-shot stepping (BASELINE config 4: 32 independent sources) on the DMMA path.

Shot q of run_shots must equal the reference semantics of a separate
CoupledStepper run with that single source, checked
against the single-source GPU stepper and the CPU oracle on shared
coefficients.
"""

import math

import numpy as np
import pytest

from helpers import face_probes, load_golden, models_from_arrays, partition_for, rel
from oracle import sfw_oracle as so
from paper_1406_6923_b200 import CoupledStepper, Probe, SourceTerm, build_models
from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200.configs import locate, make_workload

pytestmark = pytest.mark.gpu


def _shots(models, n, seed):
    rng = np.random.default_rng(seed)
    order = sorted(models)
    out = []
    for q in range(n):
        a = order[rng.integers(len(order))]
        md = models[a]
        v = rng.standard_normal(md.state_size) * 1e-6
        v[:md.width] = 0.0  # interior sources never touch the face layer (stepper.py:116-123)
        f0 = 5.0 + 10.0 * rng.random()
        out.append(SourceTerm(a, v, so.ricker(f0, 1.2 / f0)))
    return out


def test_shots_match_single_source_runs_config1():
    g = load_golden("golden_c1.npz")
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    shots = _shots(models, 32, 3)
    dt = float(g["dt"])
    n = 120
    with CoupledStepper(models, dt) as st:
        times, rows = st.run_shots(n, shots, probes=probes)
        assert rows.shape == (n + 1, 32, len(probes))
        uq = st.shot_state(5)[0]
    for q in (0, 5, 17, 31):
        with CoupledStepper(models, dt, sources=(shots[q],)) as st1:
            t1, r1 = st1.run(n, probes=probes)
            u1 = st1.u_curr
        assert np.array_equal(times, t1)
        assert rel(rows[:, q, :], r1) < 1e-10, q
        if q == 5:
            for a in u1:
                assert rel(uq[a], u1[a]) < 1e-10 or np.linalg.norm(u1[a]) < 1e-30
    # and against the CPU oracle for one shot
    om = {a: so.Model(alpha=a, lo=None, shape=None, spacing=None, modes_per_face=4, layers=m.layers, shift=0.0,
                      neighbors=m.neighbors, face_indices=(), gammas=m.gammas, gamma_hats=m.gamma_hats,
                      scales=m.scales, basis=None, c=None, mu=None) for a, m in models.items()}
    sh = shots[9]
    _, ro = so.Coupled(om, dt, sources=[(sh.alpha, sh.vector, sh.profile)]).run(
        n, probes=[(p.alpha, p.weights) for p in probes])
    assert rel(rows[:, 9, :], ro) < 1e-9


def test_shots_m9k8_physical_sources():
    wl = make_workload(4, counts=(2, 2, 2))
    ext = tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing))
    part = pg.build_partition(pg.DomainSpec(ext, wl.counts, wl.p))
    ops = [pg.assemble_subdomain_operator(part, a, wl.c_field) for a in sorted(s.alpha for s in part.subdomains)]
    rows_req = {}
    for ijk in wl.sources:
        a, r = locate(ijk, wl.counts, wl.p)
        rows_req.setdefault(a, []).append(r)
    models = build_models(ops, 9, 8, wl.shift, rows=rows_req)
    from paper_1406_6923_b200 import cfl_estimate_coupled, project_source
    from paper_1406_6923_b200.pulses import ricker
    lam, _ = cfl_estimate_coupled(models)
    dt = 0.9 * 2.0 / math.sqrt(lam)
    shots = []
    for ijk in wl.sources:
        a, r = locate(ijk, wl.counts, wl.p)
        shots.append(SourceTerm(a, project_source(models[a], r), ricker(wl.f0, wl.delay)))
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    n = 80
    with CoupledStepper(models, dt) as st:
        _, rows = st.run_shots(n, shots, probes=probes)
    # m9k8 tolerance: max(1e-9, 10 x the oracle's own summation-order floor)
    om = {a: so.Model(alpha=a, lo=None, shape=None, spacing=None, modes_per_face=9, layers=m.layers, shift=0.0,
                      neighbors=m.neighbors, face_indices=(), gammas=m.gammas, gamma_hats=m.gamma_hats,
                      scales=m.scales, basis=None, c=None, mu=None) for a, m in models.items()}
    fm = {a: so.Model(alpha=a, lo=None, shape=None, spacing=None, modes_per_face=9, layers=m.layers, shift=0.0,
                      neighbors=m.neighbors, face_indices=(), gammas=[np.asfortranarray(b) for b in m.gammas],
                      gamma_hats=[np.asfortranarray(b) for b in m.gamma_hats], scales=m.scales, basis=None,
                      c=None, mu=None) for a, m in models.items()}
    pw = [(p.alpha, p.weights) for p in probes]
    for q in (0, 13, 31):
        src = [(shots[q].alpha, shots[q].vector, shots[q].profile)]
        _, ro = so.Coupled(om, dt, sources=src).run(n, probes=pw)
        _, rf = so.Coupled(fm, dt, sources=src).run(n, probes=pw)
        tol = max(1e-9, 10 * rel(rf, ro))
        with CoupledStepper(models, dt, sources=(shots[q],)) as st1:
            _, r1 = st1.run(n, probes=probes)
        e_single, e_oracle = rel(rows[:, q, :], r1), rel(rows[:, q, :], ro)
        print(f"shot {q}: vs single-source GPU {e_single:.2e}, vs oracle {e_oracle:.2e}, tol {tol:.2e}")
        assert e_single < tol and e_oracle < tol


@pytest.mark.parametrize("maxgrid", [None, "3", "1"])
def test_shots_short_runs_and_strided_records(maxgrid, monkeypatch):
    """The layer-0 pass of step k runs inside the sweep of step k+1 and once more after the last step
    (sfw_shots.cu): 1-, 2- and 3-step runs, strided records and several subdomains per team
    (SFW_STEP_MAXGRID caps the number of teams) against the single-source stepper."""
    if maxgrid:
        monkeypatch.setenv("SFW_STEP_MAXGRID", maxgrid)
    g = load_golden("golden_c1.npz")
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    rng = np.random.default_rng(11)
    order = sorted(models)
    probes.append(Probe(order[3], rng.standard_normal(models[order[3]].state_size)))  # dense node-type weights
    shots = _shots(models, 32, 5)
    dt = float(g["dt"])
    for n, every in ((1, 1), (2, 1), (3, 1), (7, 3), (40, 4)):
        with CoupledStepper(models, dt) as st:
            times, rows = st.run_shots(n, shots, probes=probes, record_every=every)
            states = {q: st.shot_state(q) for q in (2, 30)}
        assert rows.shape == (n // every + 1, 32, len(probes))
        for q in (2, 30):
            with CoupledStepper(models, dt, sources=(shots[q],)) as st1:
                t1, r1 = st1.run(n, probes=probes, record_every=every)
                u1, p1 = st1.u_curr, st1.u_prev
            assert np.array_equal(times, t1)
            assert rel(rows[:, q, :], r1) < 1e-10 or np.abs(r1).max() < 1e-300, (n, every, q)
            big = max(np.abs(v).max() for v in u1.values())
            for a in u1:  # both time levels, layer 0 included (completed by the pass after the last step)
                assert np.abs(states[q][0][a] - u1[a]).max() <= 1e-10 * big, (n, every, q, a)
                assert np.abs(states[q][1][a] - p1[a]).max() <= 1e-10 * big, (n, every, q, a)
