"""Host-side pieces of the auxiliary rows (fine-grid solver, transfer maps) -- no GPU needed."""

import numpy as np
import pytest

from helpers import partition_for
from paper_1406_6923_b200 import ConfigError, FineGridOperator, assemble_global_operator
from paper_1406_6923_b200.configs import make_workload
from paper_1406_6923_b200.ntd import frequency_band, nudge_off_poles


def test_fine_grid_operator_descriptor():
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    a = assemble_global_operator(part, wl.c_field)
    assert isinstance(a, FineGridOperator)
    assert a.shape == tuple(part.global_shape) and a.n == wl.c_field.size
    # link scale 1 / (w * h^2), w = 1, as grid.py:366 forms it
    for s, h in zip(a.scales, part.spacing):
        assert s == 1.0 / (np.ones(1) * h ** 2)[0]
    with pytest.raises(ConfigError):
        FineGridOperator((2, 2, 2), (1.0, 1.0, 1.0), np.ones(7))


def test_frequency_band_and_pole_nudging():
    w = frequency_band(2.0, 50.0, 7)
    assert np.array_equal(w, np.geomspace(2.0, 50.0, 7))
    with pytest.raises(ConfigError):
        frequency_band(5.0, 1.0)
    with pytest.raises(ConfigError):
        frequency_band(1.0, 5.0, 0)
    poles = np.array([3.0, 10.0])
    out = nudge_off_poles(np.array([3.0, 4.0, 10.0 * (1 + 1e-9)]), poles)
    assert out[1] == 4.0
    for x in out:
        assert np.min(np.abs(poles - x)) > 1e-8 * max(x, 1.0)
    assert np.array_equal(nudge_off_poles(np.array([1.0, 2.0]), np.zeros(0)), [1.0, 2.0])


def test_verify_subdomain_needs_the_operator_matrix():
    """verify_subdomain (sim.py:703-768) rejects an operator without its host matrix before any
    device work (the GPU build itself never assembles one)."""
    from paper_1406_6923_b200 import grid as pg
    from paper_1406_6923_b200.ntd import verify_subdomain
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    op = pg.assemble_subdomain_operator(part, (0, 0, 0), wl.c_field)
    with pytest.raises(ConfigError):
        verify_subdomain(op, wl.modes_per_face, wl.shift, [10.0, 20.0])


def test_operator_csr_conversion_keeps_the_band():
    """The explicit-operator maps take scipy sparse or dense input; the CSR handed to the library
    has sorted int32 indices and the operator's half-bandwidth P^2 (natural order)."""
    from paper_1406_6923_b200 import grid as pg
    from paper_1406_6923_b200.ntd import _csr
    part = partition_for((2, 1, 1), (5, 5, 5), (2.0, 1.0, 1.0))
    op = pg.assemble_subdomain_operator(part, (0, 0, 0), np.ones((9, 5, 5)), with_matrix=True)
    rp, ci, val, n = _csr(op.matrix)
    assert n == 125 and rp.dtype == np.int32 and ci.dtype == np.int32 and rp[-1] == val.size
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert int(np.max(np.abs(rows - ci))) == 25
    rp2, ci2, val2, _ = _csr(op.matrix.toarray())
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(val, val2)
