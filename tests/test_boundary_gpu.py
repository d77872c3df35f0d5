"""Drop-in boundary pieces beyond build/step, through the C ABI on the GPU.

* project_state / state_to_nodes (reference rom.py:437-459) vs the reference's own outputs
  (golden_states.npz, tests/golden/make_golden.py golden_states);
* Interface.mass (stepper.py:64-70, 204-210): the device-computed masses vs the reference's;
* build_models refuses an operator whose explicit matrix is not the finite-volume operator of its
  (c, mu, spacing, neighbours) -- the GPU build never reads op.matrix.
"""

import dataclasses

import numpy as np
import pytest

from helpers import load_golden, partition_for, rel
from paper_1406_6923_b200 import (ConfigError, CoupledStepper, NumericalError, build_models, project_state,
                                  state_to_nodes)
from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200.configs import make_workload

pytestmark = pytest.mark.gpu


def _c1():
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    ops = [pg.assemble_subdomain_operator(part, a, wl.c_field) for a in sorted(s.alpha for s in part.subdomains)]
    return wl, part, ops


def test_project_state_and_state_to_nodes_match_reference():
    g = load_golden("golden_states.npz")
    wl, part, ops = _c1()
    a = tuple(int(x) for x in g["alpha"])
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift, basis={a})
    md = models[a]
    p = project_state(md, g["x"])
    n = state_to_nodes(md, g["u"])
    print("project_state", rel(p, g["projected"]), "state_to_nodes", rel(n, g["nodes"]))
    assert rel(p, g["projected"]) < 1e-9
    assert rel(n, g["nodes"]) < 1e-9
    # inverse pair on the reduction subspace
    assert rel(project_state(md, state_to_nodes(md, g["u"])), g["u"]) < 1e-9
    other = next(b for b in models if b != a)
    with pytest.raises(NumericalError):
        project_state(models[other], g["x"])  # built without its basis (rom.py:439-440)
    with pytest.raises(ConfigError):
        project_state(md, g["x"][:-1])


def test_interface_masses_match_reference():
    g = load_golden("golden_states.npz")
    wl, part, ops = _c1()
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift)
    with CoupledStepper(models, 1e-4) as st:
        ifs = st.interfaces
        assert len(ifs) == len(g["pairs"])
        for i, (itf, pr) in enumerate(zip(ifs, g["pairs"])):
            assert (itf.low, itf.low_face, itf.high, itf.high_face) == (tuple(pr[:3]), pr[3], tuple(pr[4:7]), pr[7])
            assert itf.mass.shape == (4, 4)
            assert rel(itf.mass, g["masses"][i]) < 1e-9
            assert np.array_equal(itf.mass, itf.mass.T)


def test_build_checks_an_explicit_operator_matrix():
    wl, part, ops = _c1()
    op = pg.assemble_subdomain_operator(part, (0, 1, 0), wl.c_field, with_matrix=True)
    assert op.matrix is not None
    md = build_models([op], wl.modes_per_face, wl.n, wl.shift)[(0, 1, 0)]
    assert md.layers == wl.n + 1
    bad = op.matrix.copy()
    bad.data = bad.data * 1.001
    with pytest.raises(ConfigError):
        build_models([dataclasses.replace(op, matrix=bad)], wl.modes_per_face, wl.n, wl.shift)


def test_state_assignment_writes_through():
    """u_curr / u_prev are mutable in the reference (stepper.py:164-165): assigning them (or an item)
    sets the device state, and stepping continues from it exactly."""
    wl, part, ops = _c1()
    models = build_models(ops, wl.modes_per_face, wl.n, wl.shift)
    rng = np.random.default_rng(11)
    u0 = {a: rng.standard_normal(m.state_size) * 1e-3 for a, m in models.items()}
    for a, m in models.items():  # shared-face replicas agree
        for f, b in m.neighbors.items():
            if b > a:
                u0[b][models[b].face_slice(f ^ 1)] = u0[a][m.face_slice(f)]
    with CoupledStepper(models, 1e-4) as st, CoupledStepper(models, 1e-4) as st2:
        st.initialize(u0)
        for _ in range(7):
            st.advance()
        uc, up = st.u_curr, st.u_prev
        st2.initialize(u0)  # same growth-detector baseline as st (stepper.py:357-360)
        st2.u_curr = dict(uc)
        view = st2.u_prev
        for a in up:
            view[a] = up[a]  # item assignment writes through
        for _ in range(5):
            st.advance()
            st2.advance()
        a_state, b_state = st.u_curr, st2.u_curr
    for a in a_state:
        assert np.array_equal(a_state[a], b_state[a])
