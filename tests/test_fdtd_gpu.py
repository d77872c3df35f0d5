"""Fine-grid leapfrog reference solver on the GPU (reference reference.py, grid.py:461-467).

The golden vectors were produced by the reference itself (make_golden.py::golden_fdtd:
assemble_global_operator + estimate_lambda_max + run_leapfrog on the config-1 grid, 33^3
nodes, 200 steps, Ricker source as sim.run_reference drives it).  The GPU stencil rebuilds the
CSR rows in the reference's arithmetic, so products and trajectories are compared bit for bit.
"""

import math

import numpy as np
import pytest

from helpers import load_golden, partition_for, rel
from oracle import sfw_oracle as so
from paper_1406_6923_b200 import (ConfigError, InstabilityError, assemble_global_operator, estimate_lambda_max,
                                  leapfrog_energy, run_leapfrog, stability_limit)
from paper_1406_6923_b200.configs import make_workload
from paper_1406_6923_b200.pulses import ricker

pytestmark = pytest.mark.gpu


def _config1():
    wl = make_workload(1)
    part = partition_for(wl.counts, wl.p, tuple((s - 1) * h for s, h in zip(wl.global_shape, wl.spacing)))
    return wl, part, assemble_global_operator(part, wl.c_field)


def test_product_bitwise_vs_reference():
    g = load_golden("golden_fdtd.npz")
    _, _, a = _config1()
    x = np.random.default_rng(3).standard_normal(a.n)
    assert np.array_equal(a @ x, g["av"])


def test_power_iteration_vs_reference():
    g = load_golden("golden_fdtd.npz")
    _, _, a = _config1()
    lam = estimate_lambda_max(a)
    assert abs(lam - float(g["lam"])) <= 1e-7 * float(g["lam"])
    assert abs(stability_limit(a) - 2.0 / math.sqrt(float(g["lam"]))) <= 1e-7 * 2.0 / math.sqrt(float(g["lam"]))


def test_forced_run_bitwise_vs_reference():
    g = load_golden("golden_fdtd.npz")
    wl, _, a = _config1()
    vec = np.zeros(a.n)
    src = int(g["src"])
    vec[src] = 1.0 / wl.c_field.ravel()[src]
    run = run_leapfrog(a, float(g["dt"]), 200, source_vec=vec, source_fn=ricker(wl.f0, wl.delay),
                       record_idx=g["rec"], record_every=1, chunk=64)
    assert np.array_equal(run.times, g["times"])
    assert np.array_equal(run.samples, g["samples"]), rel(run.samples, g["samples"])
    assert np.array_equal(run.u_curr, g["u_curr"]) and np.array_equal(run.u_prev, g["u_prev"])


def test_free_run_vs_oracle_with_velocity_damping_and_record_every():
    part = partition_for((2, 2, 1), (9, 9, 9), (1.6, 1.6, 0.8))
    shape = part.global_shape
    rng = np.random.default_rng(11)
    c = rng.uniform(1.0, 2.5, shape)
    a = assemble_global_operator(part, c)
    am = so.global_matrix(shape, part.spacing, c)
    dt = 0.8 * 2.0 / math.sqrt(so.power_lambda(am)[0])
    u0, v0 = rng.standard_normal(a.n), rng.standard_normal(a.n)
    damp = 1.0 - 1e-3 * rng.random(a.n)
    rec = [0, 5, a.n // 2, a.n - 1]
    run = run_leapfrog(a, dt, 90, u0=u0, v0=v0, record_idx=rec, record_every=7, damping=damp, chunk=20)
    s, t, up, uc = so.leapfrog(am, dt, 90, u0=u0, v0=v0, record_idx=rec, record_every=7, damping=damp)
    assert np.array_equal(run.times, t)
    assert np.array_equal(run.samples, s)
    assert np.array_equal(run.u_curr, uc) and np.array_equal(run.u_prev, up)


def test_energy_conserved_and_instability_detected():
    _, _, a = _config1()
    rng = np.random.default_rng(2)
    u0 = rng.standard_normal(a.n)
    dtm = stability_limit(a)
    run = run_leapfrog(a, 0.9 * dtm, 300, u0=u0)
    e0 = None
    run0 = run_leapfrog(a, 0.9 * dtm, 1, u0=u0)
    e0 = leapfrog_energy(a, run0.u_prev, run0.u_curr, 0.9 * dtm)
    e1 = leapfrog_energy(a, run.u_prev, run.u_curr, 0.9 * dtm)
    assert abs(e1 - e0) <= 1e-9 * abs(e0)
    with pytest.raises(InstabilityError):
        run_leapfrog(a, 1.1 * dtm, 2000, u0=u0)


def test_rejects_non_grid_operators():
    with pytest.raises(ConfigError):
        estimate_lambda_max(np.eye(3))
    with pytest.raises(ConfigError):
        run_leapfrog(lambda v: v, 0.1, 3)
