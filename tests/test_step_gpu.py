"""GPU parity of the on-line stage (CoupledStepper on sm_100a) through the C ABI.

Contract: on shared coefficients, traces agree with the reference
within rel-L2 1e-9 for m=4; for m=9,k=8 within max(1e-9, 10 x the oracle's own
summation-order floor), measured here by re-running the oracle with
Fortran-ordered chain blocks.  Bitwise run-to-run determinism and bitwise
shared-face replicas are checked as the reference's tests do
(test_stepper.py:185-194, 308-322).
"""

import math

import numpy as np
import pytest

from helpers import face_probes, load_golden, models_from_arrays, oracle_models, partition_for, rel
from oracle import sfw_oracle as so
from paper_1406_6923_b200 import (ConfigError, CoupledStepper, InstabilityError, NumericalError, Probe,
                                  ProtocolError, SourceTerm, cfl_estimate_coupled, make_probe,
                                  project_source)
from paper_1406_6923_b200.configs import locate, make_workload

pytestmark = pytest.mark.gpu


def _toy(tag):
    g = load_golden("golden_toy.npz")
    pre = tag + "_"
    counts = tuple(int(x) for x in g[pre + "counts"])
    part = partition_for(counts, (5, 5, 5), tuple(float(c) for c in counts))
    models = models_from_arrays(part, g[pre + "c_field"], int(g[pre + "m"]), g[pre + "gammas"], g[pre + "hats"],
                                g[pre + "scales"], shift=4.0, basis=g[pre + "basis"])
    return g, pre, models


@pytest.mark.parametrize("tag", ["pair", "quad"])
def test_toy_run_matches_reference_golden(tag):
    g, pre, models = _toy(tag)
    order = sorted(models)
    vec = g[pre + "src_vec"]
    pw = g[pre + "probe_w"]
    u0 = {a: g[pre + "u0"][i] for i, a in enumerate(order)}
    ricker = so.ricker(1.0, 1.2)
    with CoupledStepper(models, float(g[pre + "dt"]), sources=(SourceTerm(order[0], vec, ricker),)) as st:
        times, rows = st.run(40, probes=[Probe(order[-1], pw)], u0=u0)
        assert np.array_equal(times, g[pre + "times"])
        assert rel(rows, g[pre + "rows"]) < 1e-9
        uc, up = st.u_curr, st.u_prev
        for i, a in enumerate(order):
            assert rel(uc[a], g[pre + "u_curr"][i]) < 1e-9
            assert rel(up[a], g[pre + "u_prev"][i]) < 1e-9
        assert st.message_count == int(g[pre + "messages"])
        e = st.energy()
        assert abs(e - float(g[pre + "energy"])) <= 1e-9 * abs(float(g[pre + "energy"]))


def test_toy_maps_match_reference_golden():
    g, pre, models = _toy("quad")
    order = sorted(models)
    vec = project_source(models[order[0]], 31)
    assert rel(vec, g[pre + "src_vec"]) < 1e-12
    pr = make_probe(models[order[-1]], 31)
    assert rel(pr.weights, g[pre + "probe_w"]) < 1e-12


def test_config1_traces_match_reference_golden():
    g = load_golden("golden_c1.npz")
    wl = make_workload(1, n_steps=int(g["n_steps"]))
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    src_alpha = tuple(int(x) for x in g["src_alpha"])
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    src = SourceTerm(src_alpha, g["src_vec"], so.ricker(wl.f0, wl.delay))
    with CoupledStepper(models, float(g["dt"]), sources=(src,)) as st:
        times, rows = st.run(wl.n_steps, probes=probes)
        assert np.array_equal(times, g["times"])
        assert rel(rows, g["rows"]) < 1e-9
        assert st.message_count == int(g["message_count"])
        # determinism: a second run is bitwise identical
        times2, rows2 = st.run(wl.n_steps, probes=probes)
        assert np.array_equal(rows, rows2)
        # shared-face replicas bitwise equal (test_stepper.py:185-194)
        uc = st.u_curr
        for a in st.order:
            for f, b in models[a].neighbors.items():
                assert np.array_equal(uc[a][models[a].face_slice(f)], uc[b][models[b].face_slice(f ^ 1)])


@pytest.mark.parametrize("grid", ["1", "3"])
def test_config1_traces_with_many_subdomains_per_cta(grid, monkeypatch):
    """Force several subdomains (and layer items) per CTA so cross-warp hand-offs are exercised."""
    monkeypatch.setenv("SFW_STEP_MAXGRID", grid)
    g = load_golden("golden_c1.npz")
    wl = make_workload(1, n_steps=int(g["n_steps"]))
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    src_alpha = tuple(int(x) for x in g["src_alpha"])
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    src = SourceTerm(src_alpha, g["src_vec"], so.ricker(wl.f0, wl.delay))
    with CoupledStepper(models, float(g["dt"]), sources=(src,)) as st:
        _, rows = st.run(wl.n_steps, probes=probes)
    assert rel(rows, g["rows"]) < 1e-9


def test_config1_source_vector_matches_golden():
    g = load_golden("golden_c1.npz")
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    src_alpha, row = locate(wl.sources[0], wl.counts, wl.p)
    md = models[src_alpha]
    basis = np.zeros((int(np.prod(md.shape)), md.state_size))
    basis[row] = g["src_basis_row"]
    md.basis = basis
    assert rel(project_source(md, row), g["src_vec"]) < 1e-12


def test_cfl_estimate_matches_oracle():
    g, pre, models = _toy("quad")
    lam, conv = cfl_estimate_coupled(models)
    assert conv
    assert abs(lam - float(g[pre + "lam"])) <= 1e-8 * lam


def test_acceleration_matches_oracle():
    g, pre, models = _toy("quad")
    order = sorted(models)
    omodels = {a: so.Model(alpha=a, lo=None, shape=None, spacing=None, modes_per_face=4, layers=m.layers,
                           shift=4.0, neighbors=m.neighbors, face_indices=(), gammas=m.gammas,
                           gamma_hats=m.gamma_hats, scales=m.scales, basis=None, c=m.c, mu=m.mu)
               for a, m in models.items()}
    ref = so.Coupled(omodels, 0.01)
    rng = np.random.default_rng(4)
    states = {a: rng.standard_normal(models[a].state_size) for a in order}
    with CoupledStepper(models, 0.01) as st:
        got = st._acceleration(states)
    want = ref.acceleration(states)
    for a in order:
        assert rel(got[a], want[a]) < 1e-12


@pytest.mark.parametrize("counts,env", [
    ((2, 2, 2), {}),                                                  # SMEM-resident kernel
    ((3, 3, 3), {"SFW_NO_RESIDENT": "1"}),                            # k_ustep (one interior subdomain)
    ((2, 2, 2), {"SFW_NO_RESIDENT": "1", "SFW_NO_USTEP": "1"}),       # streamed k_step2
], ids=["resident", "ustep", "step2"])
def test_m9k8_stepping_parity_on_shared_coefficients(counts, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    wl = make_workload(3, counts=counts, n_steps=60)
    models = oracle_models(wl)
    lam, _ = so.cfl_power(models)
    dt = 0.9 * 2.0 / math.sqrt(lam)
    src_alpha, row = locate(wl.sources[0], wl.counts, wl.p)
    vec = so.source_vector(models[src_alpha], row)
    rng = np.random.default_rng(11)
    order = sorted(models)
    # face taps plus dense probes (every state entry weighted) on three subdomains
    probes = face_probes(models, wl) + [(a, rng.standard_normal(models[a].state_size))
                                        for a in (order[0], src_alpha, order[-1])]
    prof = so.ricker(wl.f0, wl.delay)
    ref_rows = so.Coupled(models, dt, sources=[(src_alpha, vec, prof)]).run(wl.n_steps, probes=probes)[1]
    # oracle's own summation-order floor: Fortran-ordered chain blocks
    fmodels = {}
    for a, md in models.items():
        import dataclasses
        fmodels[a] = dataclasses.replace(md, gammas=[np.asfortranarray(b) for b in md.gammas],
                                         gamma_hats=[np.asfortranarray(b) for b in md.gamma_hats])
    alt_rows = so.Coupled(fmodels, dt, sources=[(src_alpha, vec, prof)]).run(wl.n_steps, probes=probes)[1]
    floor = rel(alt_rows, ref_rows)
    tol = max(1e-9, 10 * floor)
    with CoupledStepper(models, dt, sources=(SourceTerm(src_alpha, vec, prof),)) as st:
        gp = [Probe(a, w) for a, w in probes]
        _, rows = st.run(wl.n_steps, probes=gp)
        _, rows3 = st.run(wl.n_steps, probes=gp, record_every=3)
    assert np.array_equal(rows3, rows[::3])  # sparse recording is the same arithmetic
    err = rel(rows, ref_rows)
    print(f"m9k8 trace rel err {err:.3e}, oracle floor {floor:.3e}")
    assert err <= tol


def test_errors_follow_reference_taxonomy():
    g, pre, models = _toy("pair")
    order = sorted(models)
    with pytest.raises(ConfigError):
        CoupledStepper(models, 0.0)
    with pytest.raises(ProtocolError):
        CoupledStepper({order[0]: models[order[0]]}, 0.01)
    import dataclasses
    bad = dict(models)
    bad[order[0]] = dataclasses.replace(models[order[0]], gamma_hats=models[order[0]].gamma_hats * 1.5)
    with pytest.raises(NumericalError):
        CoupledStepper(bad, 0.01)
    shared = int(np.nonzero(models[order[0]].mu < 1.0)[0][0])
    with pytest.raises(ConfigError):
        project_source(models[order[0]], shared)
    with pytest.raises(ConfigError):
        CoupledStepper(models, 0.01, sources=(SourceTerm((9, 9, 9), np.zeros(3), lambda t: 0.0),))


def test_instability_detected():
    g, pre, models = _toy("pair")
    order = sorted(models)
    rng = np.random.default_rng(0)
    u0 = {a: rng.standard_normal(models[a].state_size) for a in order}
    for a in order:
        for f, b in models[a].neighbors.items():
            if b > a:
                u0[b][models[b].face_slice(f ^ 1)] = u0[a][models[a].face_slice(f)]
    dt = 10.0 * 2.0 / math.sqrt(float(g[pre + "lam"]))
    with CoupledStepper(models, dt) as st:
        with pytest.raises(InstabilityError):
            st.run(400, u0=u0)
        # stops where the reference stops (stepper.py:379-389): same step, same state
        omodels = {a: so.Model(alpha=a, lo=None, shape=None, spacing=None, modes_per_face=m.modes_per_face,
                               layers=m.layers, shift=4.0, neighbors=m.neighbors, face_indices=(), gammas=m.gammas,
                               gamma_hats=m.gamma_hats, scales=m.scales, basis=None, c=m.c, mu=m.mu)
                   for a, m in models.items()}
        ref = so.Coupled(omodels, dt)
        with pytest.raises(so.OracleError) as ei:
            ref.run(400, u0=u0)
        assert ei.value.kind == "InstabilityError"
        assert 0 < st.steps_done == ref.steps_done < 400
        assert st.time == ref.time
        uc = st.u_curr
        for a in order:
            assert rel(uc[a], ref.u_curr[a]) < 1e-8


def test_advance_equals_run():
    g, pre, models = _toy("quad")
    order = sorted(models)
    u0 = {a: g[pre + "u0"][i] for i, a in enumerate(order)}
    dt = float(g[pre + "dt"])
    with CoupledStepper(models, dt) as st:
        st.initialize(u0)
        for _ in range(25):
            st.advance()
        a_state = st.u_curr
        assert st.steps_done == 25 and st.message_count == 25 * 2 * len(st.interfaces)
        st.run(25, u0=u0)
        b_state = st.u_curr
    for a in order:
        assert np.array_equal(a_state[a], b_state[a])


@pytest.mark.parametrize("record_every,env", [(1, {}), (3, {}), (1, {"SFW_NO_RESIDENT": "1", "SFW_NO_SW": "1"})],
                         ids=["resident", "record3", "streamed"])
def test_chunked_run_equals_single_launch(record_every, env, monkeypatch):
    """Large probe-row downloads split the run into chunks whose rows download while later
    chunks compute (sfw_step_run); the traces, times and final state equal one launch bit for bit."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g, pre, models = _toy("quad")
    order = sorted(models)
    u0 = {a: g[pre + "u0"][i] for i, a in enumerate(order)}
    dt = float(g[pre + "dt"])
    probes = [Probe(a, np.eye(models[a].state_size)[j]) for a in order for j in (0, 3, models[a].state_size - 1)]
    n = 203
    out = {}
    for mode in ("single", "chunked"):
        monkeypatch.setenv("SFW_NO_CHUNK" if mode == "single" else "SFW_CHUNK_BYTES", "1")
        if mode == "chunked":
            monkeypatch.delenv("SFW_NO_CHUNK")
        with CoupledStepper(models, dt) as st:
            t, r = st.run(n, probes=probes, record_every=record_every, u0=u0)
            out[mode] = (t, r, st.u_curr)
    ts, rs, us = out["single"]
    tc, rc, uc = out["chunked"]
    assert rs.shape == (1 + n // record_every, len(probes))
    assert np.array_equal(ts, tc) and np.array_equal(rs, rc)
    for a in order:
        assert np.array_equal(us[a], uc[a])


def test_start_from_rest_fast_path_is_bitwise(monkeypatch):
    """From rest the start skips the acceleration pass (acc(0) = 0); traces and state equal the
    full mode-1 start (SFW_INIT_FULL) bit for bit."""
    g = load_golden("golden_c1.npz")
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    models = models_from_arrays(part, wl.c_field, 4, g["gammas"], g["hats"], g["scales"], shift=wl.shift)
    src_alpha = tuple(int(x) for x in g["src_alpha"])
    src = SourceTerm(src_alpha, g["src_vec"], so.ricker(wl.f0, wl.delay))
    probes = [Probe(a, w) for a, w in face_probes(models, wl)]
    out = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("SFW_INIT_FULL", env)
        with CoupledStepper(models, float(g["dt"]), sources=(src,)) as st:
            _, rows = st.run(50, probes=probes)
            out.append((rows, st.u_curr, st.u_prev))
    assert np.array_equal(out[0][0], out[1][0])
    for a in out[0][1]:
        assert np.array_equal(out[0][1][a], out[1][1][a]) and np.array_equal(out[0][2][a], out[1][2][a])
