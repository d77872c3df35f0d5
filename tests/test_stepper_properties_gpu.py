"""The reference stepper's behavioural contract (pkg/tests/test_stepper.py, test_rom.py), checked on
the GPU path: structure of the chain operator, dense-leapfrog equivalence, symmetrizable negative
coupling, convergence of coupled traces to the fine grid, energy conservation, message counts,
protocol errors, worker invariance, CFL vs the dense spectrum, interlacing with the fine-grid step,
source/probe preconditions, probe vs node reconstruction, mirror symmetry, zero data.

The checks are restated here for this package's API (dimensionless unit-cube media, p = 5..12
nodes per edge, shift 4 as the reference's tests use); the dense linear algebra below is test-side
verification only.
"""

import dataclasses
import math

import numpy as np
import pytest

from oracle import sfw_oracle as so
from paper_1406_6923_b200 import (ConfigError, CoupledStepper, NumericalError, ProtocolError, SourceTerm,
                                  assemble_global_operator, build_models, build_subdomain_model,
                                  cfl_estimate_coupled, make_probe, project_source, run_leapfrog,
                                  stability_limit, stable_step_coupled, state_to_nodes)
from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200.ntd import ntd_chain
from paper_1406_6923_b200.stepper import chain_operator

pytestmark = pytest.mark.gpu


def _part(counts, p, extents=None):
    ext = tuple(float(c) for c in counts) if extents is None else extents
    return pg.build_partition(pg.DomainSpec(ext, tuple(counts), (p, p, p)))


def _models(counts=(2, 1, 1), p=5, m=1, n=2, c=None, shift=4.0):
    part = _part(counts, p)
    c = np.ones(part.global_shape) if c is None else c
    ops = {s.alpha: pg.assemble_subdomain_operator(part, s.alpha, c) for s in part.subdomains}
    models = build_models(list(ops.values()), m, n, shift, basis="all")
    return part, c, ops, models


def _replica_consistent(models, seed):
    rng = np.random.default_rng(seed)
    st = {a: rng.standard_normal(md.state_size) for a, md in models.items()}
    for a in sorted(models):
        for f, b in sorted(models[a].neighbors.items()):
            if b > a:
                st[b][models[b].face_slice(f ^ 1)] = st[a][models[a].face_slice(f)]
    return st


def test_chain_operator_structure_and_transfer_map():
    _, _, _, models = _models(counts=(1, 1, 1), m=1, n=2)
    md = models[(0, 0, 0)]
    op = chain_operator(md)
    w, L = md.width, md.layers
    g = np.zeros_like(op)
    for j in range(L):
        g[j * w:(j + 1) * w, j * w:(j + 1) * w] = md.scales[j]
    sym = np.linalg.solve(g, op @ g)  # similar to a symmetric negative semidefinite matrix
    assert np.linalg.norm(sym - sym.T) <= 1e-9 * np.linalg.norm(sym)
    assert np.linalg.eigvalsh(0.5 * (sym + sym.T)).max() <= 1e-9
    om = 0.7
    rhs = np.zeros((L * w, w))
    rhs[:w] = md.gamma_hats[0]
    top = np.linalg.solve(om * om * np.eye(L * w) + op, rhs)[:w]
    direct = ntd_chain(md.gammas, md.gamma_hats, om)
    assert np.linalg.norm(top - direct) <= 1e-9 * np.linalg.norm(direct)


def test_single_subdomain_equals_dense_leapfrog():
    _, _, _, models = _models(counts=(1, 1, 1), m=1, n=2)
    md = models[(0, 0, 0)]
    dense = chain_operator(md)
    lam = (-np.linalg.eigvals(dense).real).max()
    dt = 0.8 * 2.0 / math.sqrt(lam)
    rng = np.random.default_rng(3)
    u0, v0 = rng.standard_normal(md.state_size), rng.standard_normal(md.state_size)
    _, _, _, want = so.leapfrog(dense, dt, 60, u0=u0, v0=v0)
    with CoupledStepper(models, dt) as st:
        st.initialize({md.alpha: u0}, {md.alpha: v0})
        for _ in range(60):
            st.advance()
        got = st.u_curr[md.alpha]
        assert st.message_count == 0
    assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)


def test_coupled_acceleration_is_symmetrizable_and_negative():
    _, _, _, models = _models(m=1, n=1)
    order = sorted(models)
    # merged unknowns: a shared layer-1 face segment is one unknown, owned by the lower subdomain
    owned = {}
    for a in order:
        keep = np.ones(models[a].state_size, dtype=bool)
        for f, b in models[a].neighbors.items():
            if b < a:
                keep[models[a].face_slice(f)] = False
        owned[a] = keep
    pairs = [(a, i) for a in order for i in np.nonzero(owned[a])[0]]
    index = {pq: k for k, pq in enumerate(pairs)}

    def home(a, i):  # merged index of slot i of subdomain a (replicas map to their owner)
        if (a, i) in index:
            return index[(a, i)]
        f = next(f for f in models[a].neighbors if models[a].face_slice(f).start <= i < models[a].face_slice(f).stop)
        b = models[a].neighbors[f]
        return index[(b, models[b].face_slice(f ^ 1).start + i - models[a].face_slice(f).start)]

    size = len(pairs)
    dense = np.zeros((size, size))
    with CoupledStepper(models, dt=0.01) as st:
        for k in range(size):
            states = {a: np.zeros(models[a].state_size) for a in order}
            for a in order:
                for i in range(models[a].state_size):
                    if home(a, i) == k:
                        states[a][i] = 1.0
            acc = st._acceleration(states)
            dense[:, k] = [acc[a][i] for a, i in pairs]
    mass = np.zeros((size, size))
    for a in order:
        md = models[a]
        rows = np.array([home(a, i) for i in range(md.state_size)])
        for j in range(md.layers):
            blk = rows[j * md.width:(j + 1) * md.width]
            mass[np.ix_(blk, blk)] += np.linalg.inv(md.gamma_hats[j])
    wgt = mass @ dense
    assert np.linalg.norm(wgt - wgt.T) <= 1e-8 * np.linalg.norm(wgt)
    ev = np.linalg.eigvalsh(0.5 * (wgt + wgt.T))
    assert ev.max() <= 1e-8 * abs(ev.min())


def test_coupled_traces_converge_to_the_fine_grid():
    """Two subdomains (p = 12), a 1.3 inclusion across x in [1.2, 1.7], interior Ricker source;
    receivers across the interface: the reduced traces approach the fine-grid leapfrog ones as
    the number of inverse moments grows (reference test_stepper.py:197-258)."""
    p = 12
    part = _part((2, 1, 1), p, extents=(2.0, 1.0, 1.0))
    gs = part.global_shape
    c = np.ones(gs)
    xs = [np.arange(g) * h for g, h in zip(gs, part.spacing)]
    box = np.ix_(*[(x >= lo) & (x <= hi) for x, lo, hi in zip(xs, (1.2, 0.3, 0.3), (1.7, 0.8, 0.8))])
    c[box] = 1.3
    ops = {s.alpha: pg.assemble_subdomain_operator(part, s.alpha, c) for s in part.subdomains}
    f0, t0 = 0.75, 1.2 / 0.75

    def pulse(t):
        arg = (math.pi * f0 * (t - t0)) ** 2
        return (1.0 - 2.0 * arg) * math.exp(-arg)

    src_ijk, rec_ijk = (6, 6, 6), [(18, 6, 6), (19, 5, 6)]
    glob = assemble_global_operator(part, c)
    src = int(np.ravel_multi_index(src_ijk, gs))
    recs = [int(np.ravel_multi_index(r, gs)) for r in rec_ijk]
    vec = np.zeros(glob.n)
    vec[src] = 1.0 / c[src_ijk]
    dt = 0.9 * stability_limit(glob)
    n_steps = int(math.ceil(3.2 / dt))
    fine = run_leapfrog(glob, dt, n_steps, source_vec=vec, source_fn=pulse, record_idx=recs)
    want = fine.samples * np.array([c.ravel()[i] for i in recs])
    errs = []
    for n in (1, 2, 3, 4):
        models = build_models(list(ops.values()), 9, n, 4.0, basis="all")
        s = SourceTerm((0, 0, 0), project_source(models[(0, 0, 0)], ops[(0, 0, 0)].local_index(src_ijk)), pulse)
        probes = [make_probe(models[(1, 0, 0)], ops[(1, 0, 0)].local_index(r)) for r in rec_ijk]
        with CoupledStepper(models, dt, sources=[s]) as st:
            _, rows = st.run(n_steps, probes=probes)
        errs.append(float(np.linalg.norm(rows - want) / np.linalg.norm(want)))
    print("coupled vs fine-grid trace errors, n = 1..4:", errs)
    assert errs[-1] < 0.02 and errs[-1] < 0.05 * errs[0]
    assert all(b < a for a, b in zip(errs, errs[1:]))


def test_energy_conserved_step_by_step():
    _, _, _, models = _models(m=4, n=2)
    dt = 0.5 * stable_step_coupled(models)[0]
    e = []
    with CoupledStepper(models, dt) as st:
        st.initialize(_replica_consistent(models, 1), _replica_consistent(models, 2))
        for _ in range(400):
            st.advance()
            e.append(st.energy())
    e = np.array(e)
    assert e[0] > 0 and (e.max() - e.min()) / e.mean() < 1e-9


def test_message_counts_and_protocol_errors():
    _, _, _, models = _models(counts=(2, 2, 1), m=1, n=1)
    with CoupledStepper(models, dt=0.01) as st:
        assert len(st.interfaces) == 4
        with pytest.raises(ProtocolError):
            st.advance()  # not initialised
        st.initialize()
        assert st.message_count == 0
        for _ in range(7):
            st.advance()
        assert st.message_count == 7 * 8
        for a in models:  # zero data stays zero
            assert np.all(st.u_curr[a] == 0.0)
    with pytest.raises(ProtocolError):  # a neighbour without a model
        CoupledStepper({(0, 0, 0): models[(0, 0, 0)]}, dt=0.01)
    part = _part((2, 1, 1), 5)
    c = np.ones(part.global_shape)
    op0 = pg.assemble_subdomain_operator(part, (0, 0, 0), c)
    op1 = pg.assemble_subdomain_operator(part, (1, 0, 0), c)
    mixed = {(0, 0, 0): build_subdomain_model(op0, 1, 1, 4.0), (1, 0, 0): build_subdomain_model(op1, 4, 1, 4.0)}
    with pytest.raises(ProtocolError):  # mode counts differ across the shared face
        CoupledStepper(mixed, dt=0.01)


def test_workers_do_not_change_results():
    _, _, _, models = _models(counts=(2, 2, 1), m=4, n=2)
    dt = 0.4 * stable_step_coupled(models)[0]
    probes = [make_probe(models[(0, 0, 0)], 31)]
    u0 = _replica_consistent(models, 5)
    runs = []
    for workers in (1, 2, 4):
        with CoupledStepper(models, dt, workers=workers) as st:
            t, r = st.run(50, probes=probes, u0=u0)
            runs.append((t, r, st.message_count))
    for t, r, mc in runs[1:]:
        assert np.array_equal(t, runs[0][0]) and np.array_equal(r, runs[0][1]) and mc == runs[0][2]


def test_cfl_estimate_against_the_dense_spectrum():
    _, _, _, models = _models(m=1, n=1)
    order = sorted(models)
    sizes = [models[a].state_size for a in order]
    cols = []
    with CoupledStepper(models, dt=1.0) as st:
        for ia, a in enumerate(order):
            for i in range(sizes[ia]):
                states = {b: np.zeros(models[b].state_size) for b in order}
                states[a][i] = 1.0
                acc = st._acceleration(states)
                cols.append(np.concatenate([acc[b] for b in order]))
    lam_true = (-np.linalg.eigvals(np.array(cols).T).real).max()
    lam, conv = cfl_estimate_coupled(models)
    assert conv and abs(lam - lam_true) <= 1e-4 * lam_true


def test_reduced_step_is_no_shorter_than_the_fine_step():
    part = _part((1, 1, 1), 6)
    c = np.ones(part.global_shape)
    op = pg.assemble_subdomain_operator(part, (0, 0, 0), c)
    md = build_subdomain_model(op, 4, 2, 4.0)
    dt_fine = stability_limit(assemble_global_operator(part, c))  # one subdomain: the same operator
    dt_rom, _, conv = stable_step_coupled({md.alpha: md})
    assert conv and dt_rom >= dt_fine * (1.0 - 1e-9)  # Galerkin projection: interlacing spectrum


def test_source_and_probe_preconditions():
    _, _, ops, models = _models(m=1, n=1)
    md = models[(0, 0, 0)]
    with pytest.raises(ConfigError):
        project_source(md, int(np.nonzero(md.mu < 1.0)[0][0]))  # interface node
    bare = dataclasses.replace(md, basis=None, basis_rows=None)
    with pytest.raises(NumericalError):
        project_source(bare, 31)
    with pytest.raises(NumericalError):
        make_probe(bare, 31)


def test_probe_equals_node_reconstruction():
    _, _, _, models = _models(counts=(1, 1, 1), m=4, n=2)
    md = models[(0, 0, 0)]
    u = np.random.default_rng(9).standard_normal(md.state_size)
    row = 31
    via_nodes = state_to_nodes(md, u)[row] * md.c[row] / math.sqrt(md.mu[row])
    assert abs(make_probe(md, row).weights @ u - via_nodes) <= 1e-10 * max(1.0, abs(via_nodes))


def test_mirror_symmetric_receivers_record_the_same_trace():
    part = _part((2, 1, 1), 7, extents=(2.0, 1.0, 1.0))
    c = np.ones(part.global_shape)
    ops = {s.alpha: pg.assemble_subdomain_operator(part, s.alpha, c) for s in part.subdomains}
    models = build_models(list(ops.values()), 4, 2, 4.0, basis="all")

    def pulse(t):
        return math.sin(6.0 * t) * math.exp(-8.0 * (t - 0.8) ** 2)

    s = SourceTerm((0, 0, 0), project_source(models[(0, 0, 0)], ops[(0, 0, 0)].local_index((3, 3, 3))), pulse)
    probes = [make_probe(models[(1, 0, 0)], ops[(1, 0, 0)].local_index(r)) for r in ((8, 2, 3), (8, 4, 3))]
    dt = 0.8 * stable_step_coupled(models)[0]
    with CoupledStepper(models, dt, sources=[s]) as st:
        _, rows = st.run(60, probes=probes)
    assert np.abs(rows[:, 0] - rows[:, 1]).max() <= 1e-7 * max(np.abs(rows).max(), 1e-300)
