"""Pin the CPU oracle (oracle/sfw_oracle.py) against reference-generated golden vectors.

The fixtures were produced by tests/golden/make_golden.py from the real
reference package; the oracle must reproduce them (same numpy/scipy calls,
same order) to within 1e-12 relative -- in practice bitwise.
"""

import math
import os

import numpy as np
import pytest

from oracle import sfw_oracle as so
from paper_1406_6923_b200.configs import locate, make_workload

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _spacing(counts, p, extents):
    gs = so.global_shape(counts, p)
    return tuple(e / (g - 1) for e, g in zip(extents, gs))


@pytest.mark.parametrize("tag", ["pair", "quad"])
def test_toy_models_and_run(tag):
    g = np.load(os.path.join(GOLD, "golden_toy.npz"))
    pre = tag + "_"
    counts = tuple(int(x) for x in g[pre + "counts"])
    m, n = int(g[pre + "m"]), int(g[pre + "n"])
    ops = so.make_subops(counts, (5, 5, 5), _spacing(counts, (5, 5, 5), tuple(map(float, counts))),
                         g[pre + "c_field"])
    order = sorted(ops)
    assert np.allclose(ops[order[0]].matrix.toarray(), g[pre + "matrix0"], rtol=0, atol=1e-13)
    models = {a: so.build_model(ops[a], m, n, 4.0) for a in order}
    for i, a in enumerate(order):
        assert rel(models[a].gammas, g[pre + "gammas"][i]) < 1e-12
        assert rel(models[a].gamma_hats, g[pre + "hats"][i]) < 1e-12
        assert rel(models[a].scales, g[pre + "scales"][i]) < 1e-12
        assert rel(models[a].tdiag, g[pre + "tdiag"][i]) < 1e-12
        assert rel(models[a].toff, g[pre + "toff"][i]) < 1e-12
        assert rel(models[a].basis, g[pre + "basis"][i]) < 1e-12
    lam, conv = so.cfl_power(models)
    assert conv and abs(lam - float(g[pre + "lam"])) <= 1e-12 * lam
    vec = so.source_vector(models[order[0]], 31)
    assert rel(vec, g[pre + "src_vec"]) < 1e-12
    pw = so.probe_weights(models[order[-1]], 31)
    assert rel(pw, g[pre + "probe_w"]) < 1e-12
    dt = float(g[pre + "dt"])
    u0 = {a: g[pre + "u0"][i] for i, a in enumerate(order)}
    st = so.Coupled(models, dt, sources=[(order[0], vec, so.ricker(1.0, 1.2))])
    times, rows = st.run(40, probes=[(order[-1], pw)], u0=u0, v0=None)
    assert np.array_equal(times, g[pre + "times"])
    assert rel(rows, g[pre + "rows"]) < 1e-11
    assert st.message_count == int(g[pre + "messages"])
    assert abs(st.energy() - float(g[pre + "energy"])) <= 1e-10 * abs(float(g[pre + "energy"]))


def test_config1_models_traces():
    g = np.load(os.path.join(GOLD, "golden_c1.npz"))
    wl = make_workload(1, n_steps=int(g["n_steps"]))
    assert np.array_equal(wl.c_field, g["c_field"])
    ops = so.make_subops(wl.counts, wl.p, wl.spacing, wl.c_field)
    order = sorted(ops)
    models = {a: so.build_model(ops[a], wl.modes_per_face, wl.n, wl.shift) for a in order}
    for i, a in enumerate(order):
        assert rel(models[a].gammas, g["gammas"][i]) < 1e-12
        assert rel(models[a].tdiag, g["tdiag"][i]) < 1e-12
        assert rel(models[a].toff, g["toff"][i]) < 1e-12
    lam, conv = so.cfl_power(models)
    assert abs(lam - float(g["lam"])) <= 1e-12 * lam
    dt = 0.9 * 2.0 / math.sqrt(lam)
    src_alpha, src_row = locate(wl.sources[0], wl.counts, wl.p)
    vec = so.source_vector(models[src_alpha], src_row)
    assert rel(vec, g["src_vec"]) < 1e-12
    probes = []
    for alpha, face in wl.face_receivers:
        for q in range(wl.modes_per_face):
            wts = np.zeros(models[alpha].state_size)
            wts[face * wl.modes_per_face + q] = 1.0
            probes.append((alpha, wts))
    st = so.Coupled(models, dt, sources=[(src_alpha, vec, so.ricker(wl.f0, wl.delay))])
    times, rows = st.run(wl.n_steps, probes=probes)
    assert rel(rows, g["rows"]) < 1e-11
    assert st.message_count == int(g["message_count"])


def test_m9k8_subdomain_build():
    g = np.load(os.path.join(GOLD, "golden_m9k8.npz"))
    wl = make_workload(3, counts=(3, 3, 3))
    assert np.array_equal(wl.c_field, g["c_field"])
    alphas = [tuple(int(x) for x in a) for a in g["alphas"]]
    ops = so.make_subops(wl.counts, wl.p, wl.spacing, wl.c_field, alphas=alphas)
    for i, a in enumerate(alphas):
        md = so.build_model(ops[a], 9, 8, wl.shift)
        assert rel(md.tdiag, g["tdiag"][i]) < 1e-12
        assert rel(md.toff, g["toff"][i]) < 1e-12
        # bitwise with single-threaded OpenBLAS; 1e-9 is the SURVEY 8c parity bar
        assert rel(md.gammas, g["gammas"][i]) < 1e-9
        assert rel(md.gamma_hats, g["hats"][i]) < 1e-9
        assert rel(md.scales, g["scales"][i]) < 1e-9


def test_oracle_fine_grid_solver_pinned():
    """Oracle restatement of grid.py:461-467 + reference.py:26-157 vs the reference's own outputs."""
    g = np.load(os.path.join(GOLD, "golden_fdtd.npz"))
    wl = make_workload(1)
    a = so.global_matrix(wl.global_shape, wl.spacing, wl.c_field)
    x = np.random.default_rng(3).standard_normal(a.shape[0])
    assert np.array_equal(a @ x, g["av"])
    lam, _ = so.power_lambda(a)
    assert lam == float(g["lam"])
    src = int(g["src"])
    vec = np.zeros(a.shape[0])
    vec[src] = 1.0 / wl.c_field.ravel()[src]
    s, t, up, u = so.leapfrog(a, float(g["dt"]), 200, source_vec=vec, source_fn=so.ricker(wl.f0, wl.delay),
                              record_idx=g["rec"])
    assert np.array_equal(s, g["samples"]) and np.array_equal(u, g["u_curr"]) and np.array_equal(up, g["u_prev"])


def _golden_c1_models():
    g = np.load(os.path.join(GOLD, "golden_c1.npz"))
    wl = make_workload(1, n_steps=int(g["n_steps"]))
    ops = so.make_subops(wl.counts, wl.p, wl.spacing, wl.c_field)
    order = sorted(ops)
    return g, wl, {a: so.build_model(ops[a], wl.modes_per_face, wl.n, wl.shift) for a in order}


def test_batched_oracle_pinned_to_coupled():
    """oracle.CoupledBatched (full-size windows) vs the per-subdomain restatement and the
    reference's own config-1 traces; also a random-start run (every face exchanged)."""
    g, wl, models = _golden_c1_models()
    order = sorted(models)
    idx = {a: i for i, a in enumerate(order)}
    nbr = np.full((len(order), 6), -1)
    for a in order:
        for f, b in models[a].neighbors.items():
            nbr[idx[a], f] = idx[b]
    G = np.stack([models[a].gammas for a in order])
    H = np.stack([models[a].gamma_hats for a in order])
    dt = float(g["dt"])
    src_alpha, src_row = locate(wl.sources[0], wl.counts, wl.p)
    vec = so.source_vector(models[src_alpha], src_row)
    probes = []
    for alpha, face in wl.face_receivers:
        for q in range(wl.modes_per_face):
            wts = np.zeros(models[alpha].state_size)
            wts[face * wl.modes_per_face + q] = 1.0
            probes.append((alpha, wts))
    pr = so.ricker(wl.f0, wl.delay)
    bt = so.CoupledBatched(G, H, nbr, wl.modes_per_face, dt, sources=[(idx[src_alpha], vec, pr)])
    _, rows = bt.run(wl.n_steps, probes=[(idx[a], w) for a, w in probes])
    assert rel(rows, g["rows"]) < 1e-12
    rng = np.random.default_rng(4)
    u0 = rng.standard_normal(G.shape[:2] + (G.shape[2],))
    st = so.Coupled(models, dt)
    st.initialize(u0={a: u0[idx[a]].reshape(-1) for a in order})
    bt2 = so.CoupledBatched(G, H, nbr, wl.modes_per_face, dt)
    bt2.initialize(u0=u0)
    for _ in range(20):
        st.advance()
        bt2.advance()
    ref = np.stack([st.u_curr[a] for a in order])
    assert rel(bt2.u_curr.reshape(ref.shape), ref) < 1e-13


def test_golden_c2_subset_build_and_cfl():
    """golden_c2.npz (the real reference on all 512 config-2 subdomains): the oracle reproduces
    the stored inclusion-cut / source subdomains and the reference's lambda equals the GPU-independent
    value recorded with it."""
    g = np.load(os.path.join(GOLD, "golden_c2.npz"))
    wl = make_workload(2)
    alphas = [tuple(int(x) for x in a) for a in g["sub_alphas"]]
    assert len(alphas) >= 20 and g["rows"].shape == (1001, 264)
    cut = [a for a in alphas if np.any(wl.c_field[16 * a[0]:16 * a[0] + 17, 16 * a[1]:16 * a[1] + 17,
                                                   16 * a[2]:16 * a[2] + 17] == 5000.0)]
    assert len(cut) >= 8
    pick = [cut[0], cut[len(cut) // 2], tuple(int(x) for x in g["src_alpha"])]
    ops = so.make_subops(wl.counts, wl.p, wl.spacing, wl.c_field, alphas=pick)
    for a in pick:
        i = alphas.index(a)
        md = so.build_model(ops[a], 4, 6, wl.shift)
        assert rel(md.tdiag, g["sub_tdiag"][i]) < 1e-12
        assert rel(md.toff, g["sub_toff"][i]) < 1e-12
        assert rel(md.gammas, g["sub_gammas"][i]) < 1e-12
        assert rel(md.gamma_hats, g["sub_hats"][i]) < 1e-12
    src_alpha, src_row = locate(wl.sources[0], wl.counts, wl.p)
    md = so.build_model(ops[src_alpha], 4, 6, wl.shift)
    assert rel(so.source_vector(md, src_row), g["src_vec"]) < 1e-12
    assert float(g["dt"]) == 0.9 * 2.0 / math.sqrt(float(g["lam"]))


def test_golden_c5_medium_and_build():
    """golden_c5.npz: the seeded config-5 medium regenerates the stored c slices bit for bit, and the
    oracle reproduces the reference's m9k8 chain of an inclusion-cut and the source subdomain."""
    g = np.load(os.path.join(GOLD, "golden_c5.npz"))
    wl = make_workload(5)
    alphas = [tuple(int(x) for x in a) for a in g["alphas"]]
    for i, a in enumerate(alphas):
        sl = wl.c_field[16 * a[0]:16 * a[0] + 17, 16 * a[1]:16 * a[1] + 17, 16 * a[2]:16 * a[2] + 17]
        assert np.array_equal(sl, g["c_slices"][i])
    assert any(np.any(s == 5500.0) and not np.all(s == 5500.0) for s in g["c_slices"])
    pick = [alphas[-1], alphas[4]]
    ops = so.make_subops(wl.counts, wl.p, wl.spacing, wl.c_field, alphas=pick)
    for a in pick:
        i = alphas.index(a)
        md = so.build_model(ops[a], 9, 8, wl.shift)
        assert rel(md.tdiag, g["tdiag"][i]) < 1e-12
        assert rel(md.toff, g["toff"][i]) < 1e-12
        assert rel(md.gammas, g["gammas"][i]) < 1e-9
