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
