"""Fine-grid leapfrog reference solver on the GPU (mirror of reference reference.py).

The reference integrates ``w_tt = A w + f(t) s`` on the undecomposed grid with
``A = assemble_global_operator(partition, c)`` (grid.py:461-467, a scipy CSR
of ``C Lap_h C`` with mirror closure) and uses the same helpers for the CFL
estimate.  Here ``assemble_global_operator`` returns a :class:`FineGridOperator`
-- shape, spacing and ``c`` only -- and every operation runs in
``libsfw_b200.so`` (``sfw_fdtd_*``, csrc/sfw_fdtd.cu): the stencil rebuilds each
CSR row from ``c`` in the reference's arithmetic, so ``a @ x``, the power
iteration's iterates and the leapfrog trajectory match scipy/numpy bit for bit
(tests/test_fdtd_gpu.py).  There is no CPU path.

Names, arguments, defaults and errors follow reference.py:20-168:
``POWER_TOL``, ``POWER_MAX_ITER``, ``CFL_SAFETY``, ``GROWTH_LIMIT``,
``estimate_lambda_max``, ``stability_limit``, ``LeapfrogRun``, ``run_leapfrog``,
``leapfrog_energy``.
"""

from __future__ import annotations

import ctypes as C
import logging
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, InstabilityError, NumericalError

log = logging.getLogger(__name__)

POWER_TOL = 1e-8
POWER_MAX_ITER = 10000
CFL_SAFETY = 0.9
GROWTH_LIMIT = 1e6


class FineGridOperator:
    """Matrix-free ``C Lap_h C`` on a full grid (reference grid.py:461-467), applied on the GPU.

    ``a @ x`` (host vectors) returns ``A x`` exactly as the reference CSR product does.
    """

    def __init__(self, shape, spacing, c):
        self.shape = tuple(int(s) for s in shape)
        self.spacing = tuple(float(h) for h in spacing)
        self.c = np.ascontiguousarray(np.asarray(c, dtype=np.float64).ravel())
        if self.c.size != int(np.prod(self.shape)):
            raise ConfigError(f"c has {self.c.size} values for a {self.shape} grid")
        # link scale 1 / (w * h_d**2) with w = 1 (grid.py:366), formed as the reference forms it
        self.scales = np.array([float(1.0 / (np.ones(1) * h ** 2)[0]) for h in self.spacing])
        self._h = None
        self._lib = None

    @property
    def n(self) -> int:
        return self.c.size

    def _handle(self):
        if self._h is None:
            lib = _lib.load()
            h = C.c_void_p()
            eb = _lib.errbuf()
            _lib.check(lib.sfw_fdtd_create(*self.shape, _lib.dptr(self.scales), _lib.dptr(self.c), C.byref(h),
                                           eb, 1024), eb, "sfw_fdtd_create")
            self._h, self._lib = h, lib
        return self._h

    def matvec(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ConfigError(f"vector of length {x.shape} for an operator of size {self.n}")
        y = np.empty(self.n)
        eb = _lib.errbuf()
        h = self._handle()
        _lib.check(self._lib.sfw_fdtd_apply(h, _lib.dptr(x), _lib.dptr(y), eb, 1024), eb, "sfw_fdtd_apply")
        return y

    def __matmul__(self, x):
        return self.matvec(x)

    def close(self):
        if self._h is not None:
            self._lib.sfw_fdtd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _grid_op(op) -> FineGridOperator:
    if not isinstance(op, FineGridOperator):
        raise ConfigError("the GPU fine-grid solver takes the FineGridOperator of assemble_global_operator "
                          "(no CPU path for general matrices or callables)")
    return op


def estimate_lambda_max(op, n: int | None = None, *, tol: float = POWER_TOL, max_iter: int = POWER_MAX_ITER,
                        seed: int = 0) -> float:
    """Largest eigenvalue of ``-A`` by power iteration (reference.py:26-63), iterated on the GPU.

    The start vector is ``default_rng(seed).standard_normal(n)`` normalised on
    the host, as the reference draws it; non-convergence is logged and the last
    estimate returned.
    """
    a = _grid_op(op)
    if n is not None and n != a.n:
        raise ConfigError(f"state dimension {n} does not match the operator ({a.n})")
    v = np.random.default_rng(seed).standard_normal(a.n)
    v /= np.linalg.norm(v)
    lam = C.c_double()
    its = C.c_int()
    eb = _lib.errbuf()
    h = a._handle()
    _lib.check(a._lib.sfw_fdtd_power(h, _lib.dptr(v), float(tol), int(max_iter), C.byref(lam), C.byref(its), eb,
                                     1024), eb, "sfw_fdtd_power")
    if its.value < 0:
        log.warning("power iteration hit %d iterations without tol %.1e", max_iter, tol)
    estimate_lambda_max.last_iterations = abs(its.value)
    return float(lam.value)


def stability_limit(op, n: int | None = None, **kw) -> float:
    """Largest stable leapfrog step ``2 / sqrt(lambda_max(-A))`` (reference.py:66-71)."""
    lam = estimate_lambda_max(op, n, **kw)
    if lam <= 0.0:
        raise NumericalError("operator has no negative spectrum; no CFL limit")
    return 2.0 / np.sqrt(lam)


@dataclass
class LeapfrogRun:
    """Result of a leapfrog integration in the stored (symmetrized) field (reference.py:74-83)."""

    samples: np.ndarray
    times: np.ndarray
    u_prev: np.ndarray
    u_curr: np.ndarray
    dt: float
    steps: int
    kernel_ms: float = 0.0


def run_leapfrog(a, dt: float, n_steps: int, *, u0=None, v0=None, source_vec=None, source_fn=None, record_idx=None,
                 record_every: int = 1, damping=None, growth_limit: float = GROWTH_LIMIT,
                 chunk: int = 256) -> LeapfrogRun:
    """Central-difference integration of ``w_tt = A w + f(t) source_vec`` (reference.py:86-157) on the GPU.

    Records ``u[record_idx]`` at t = 0 and after every ``record_every`` steps;
    raises :class:`InstabilityError` when ``|u|`` exceeds ``growth_limit`` times
    the legitimate response scale (initial data plus the accumulated forcing).
    Steps run ``chunk`` at a time between growth checks.
    """
    op = _grid_op(a)
    n = op.n
    if record_every < 1:
        raise ConfigError("record_every must be >= 1")
    u_curr = None if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)  # None: from rest
    vel = None if v0 is None else np.ascontiguousarray(v0, dtype=np.float64)
    forced = source_vec is not None and source_fn is not None
    if forced:
        sv = np.asarray(source_vec, dtype=np.float64)
        s_idx = np.ascontiguousarray(np.flatnonzero(sv), dtype=np.int64)
        s_val = np.ascontiguousarray(sv[s_idx])
        src_norm = float(np.linalg.norm(sv))
    else:
        s_idx = np.zeros(0, np.int64)
        s_val = np.zeros(0)
        src_norm = 0.0
    rec = None if record_idx is None else np.ascontiguousarray(np.asarray(record_idx, dtype=np.int64).ravel())
    n_rec = 0 if rec is None else rec.size
    damp = None if damping is None else np.ascontiguousarray(damping, dtype=np.float64)
    h = op._handle()
    lib = op._lib
    eb = _lib.errbuf()
    _lib.check(lib.sfw_fdtd_setup(h, int(s_idx.size), _lib.lptr(s_idx), _lib.dptr(s_val), n_rec, _lib.lptr(rec),
                                  _lib.dptr(damp), eb, 1024), eb, "sfw_fdtd_setup")
    f0 = float(source_fn(0.0)) if forced else 0.0
    _lib.check(lib.sfw_fdtd_init(h, float(dt), _lib.dptr(u_curr), _lib.dptr(vel), f0, eb, 1024), eb,
               "sfw_fdtd_init")
    samples, times = [], []
    if rec is not None:
        samples.append(u_curr[rec].copy() if u_curr is not None else np.zeros(n_rec))
        times.append(0.0)
    baseline = (float(np.linalg.norm(u_curr)) if u_curr is not None else 0.0) + \
        dt * float(np.linalg.norm(vel if vel is not None else np.zeros(1)))
    step_chunk = record_every * max(1, int(chunk) // record_every)
    done = 0
    ms_total = 0.0
    while done < n_steps:
        k = min(step_chunk, n_steps - done)
        ts = [(done + i) * dt for i in range(k)]  # t_curr = (step - 1) dt, step = done + 1 + i
        prof = np.ascontiguousarray([float(source_fn(t)) for t in ts]) if forced else np.zeros(k)
        norms = np.empty(k)
        nrec = k // record_every
        rows = np.empty((max(nrec, 1), max(n_rec, 1)))
        ms = C.c_float(0.0)
        _lib.check(lib.sfw_fdtd_run(h, float(dt), int(k), _lib.dptr(prof), int(record_every), _lib.dptr(norms),
                                    _lib.dptr(rows) if n_rec else None, C.byref(ms), eb, 1024), eb, "sfw_fdtd_run")
        ms_total += ms.value
        for i in range(k):
            step = done + 1 + i
            if forced:
                baseline += dt * dt * abs(float(prof[i])) * src_norm
            nrm = float(np.sqrt(norms[i]))
            if not nrm <= growth_limit * max(baseline, 1e-300):
                raise InstabilityError(f"leapfrog diverged at step {step}: |u| = {nrm:.3e} "
                                       f"exceeds {growth_limit:.0e} x reference {baseline:.3e}")
        if rec is not None:
            for r in range(nrec):
                samples.append(rows[r, :n_rec].copy())
                times.append((done + (r + 1) * record_every) * dt)
        done += k
    uc = np.empty(n)
    up = np.empty(n)
    _lib.check(lib.sfw_fdtd_state(h, _lib.dptr(uc), _lib.dptr(up), eb, 1024), eb, "sfw_fdtd_state")
    return LeapfrogRun(samples=np.array(samples) if samples else np.zeros((0, 0)), times=np.array(times), u_prev=up,
                       u_curr=uc, dt=dt, steps=n_steps, kernel_ms=ms_total)


def leapfrog_energy(a, u_prev: np.ndarray, u_curr: np.ndarray, dt: float) -> float:
    """Discrete energy conserved by the scheme (reference.py:160-168), ``A`` applied on the GPU."""
    op = _grid_op(a)
    v = (u_curr - u_prev) / dt
    return 0.5 * float(v @ v) + 0.5 * float(u_curr @ (-(op @ u_prev)))
