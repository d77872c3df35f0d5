"""Coupled explicit leapfrog of the S-fraction ROMs -- host mirror of reference stepper.py.

Same public surface as ``sfwave.stepper`` (stepper.py:37-510): ``SourceTerm``,
``Probe``, ``Interface``, ``CoupledStepper`` (initialize / advance / run /
energy / u_curr / u_prev / message_count / steps_done / time / close),
``project_source``, ``make_probe``, ``cfl_estimate_coupled``,
``stable_step_coupled``.  All arithmetic runs in libsfw_b200.so on the GPU:
one persistent sm_100a kernel advances every subdomain for all requested
steps (csrc/sfw_step.cu); this module only marshals models, source profiles
(host callables, evaluated into a table) and bookkeeping counters.
"""

from __future__ import annotations

import ctypes as C
import logging
import operator
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .errors import ConfigError, InstabilityError, NumericalError, ProtocolError
from .rom import SubdomainModel, basis_row

log = logging.getLogger(__name__)

Alpha = tuple[int, int, int]

# reference.py:20-23 (re-exported by stepper.py:29)
POWER_TOL = 1e-8
POWER_MAX_ITER = 10000
CFL_SAFETY = 0.9
GROWTH_LIMIT = 1e6


def opposite_face(face: int) -> int:
    return face ^ 1


@dataclass(frozen=True)
class FaceMessage:
    """One face's outgoing flux slice for one step (stepper.py:37-44).

    On the GPU the messages are slices of a global face buffer written and read
    inside the stepping kernel; this type documents the protocol."""

    sender: Alpha
    face: int
    step: int
    payload: np.ndarray


@dataclass(frozen=True)
class SourceTerm:
    """Additive forcing: profile(t) times a fixed state-space vector (stepper.py:47-53)."""

    alpha: Alpha
    vector: np.ndarray
    profile: Callable[[float], float]


@dataclass(frozen=True)
class Probe:
    """Linear functional of one subdomain's state (stepper.py:56-61)."""

    alpha: Alpha
    weights: np.ndarray


@dataclass(frozen=True)
class Interface:
    """Shared face (stepper.py:64-70).  ``mass`` = (inv(Ghat_low|f) + inv(Ghat_high|f))^-1, computed
    on the device at create (ha (ha + hb)^-1 hb, symmetrised, stepper.py:204-210) and copied back."""

    low: Alpha
    low_face: int
    high: Alpha
    high_face: int
    mass: np.ndarray | None = None


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def project_source(model: SubdomainModel, local_row: int, amplitude: float = 1.0) -> np.ndarray:
    """State-space forcing of a point source at a strictly interior node (stepper.py:91-128)."""
    brow = basis_row(model, local_row)
    if model.mu[local_row] < 1.0:
        raise ConfigError(
            "source node lies on a subdomain interface (ambiguous ownership); "
            "move it strictly inside one subdomain")
    lib = _lib.load()
    L, w = model.layers, model.width
    out = np.empty(L * w)
    norms = np.zeros(2)
    eb = _lib.errbuf()
    node_norm = abs(amplitude / model.c[local_row])
    rc = lib.sfw_source_vector(L, w, _lib.dptr(_f64(model.scales)), _lib.dptr(_f64(brow)),
                               float(amplitude / model.c[local_row]), _lib.dptr(out), _lib.dptr(norms), eb, 1024)
    _lib.check(rc, eb, "project_source")
    if norms[0] <= 1e-12 * node_norm:
        log.warning("source at local node %d of subdomain %s is nearly orthogonal to the reduction "
                    "space; it will be silent", local_row, model.alpha)
    if norms[1] > 1e-8 * max(norms[0], 1e-300):
        raise NumericalError("interior source leaked into the boundary layer block "
                             f"(norm {norms[1]:.2e}); the reduction basis is inconsistent")
    return out


def make_probe(model: SubdomainModel, local_row: int) -> Probe:
    """Receiver functional returning the physical field at a local node (stepper.py:131-141)."""
    brow = basis_row(model, local_row)
    lib = _lib.load()
    L, w = model.layers, model.width
    out = np.empty(L * w)
    eb = _lib.errbuf()
    scale = float(model.c[local_row] / np.sqrt(model.mu[local_row]))
    rc = lib.sfw_probe_weights(L, w, _lib.dptr(_f64(model.scales)), _lib.dptr(_f64(brow)),
                               scale, _lib.dptr(out), eb, 1024)
    _lib.check(rc, eb, "make_probe")
    return Probe(alpha=model.alpha, weights=out)


class _StateView(dict):
    """dict of a stepper's time level whose item assignment writes through to the device."""

    def __init__(self, stepper, level, data):
        super().__init__(data)
        self._stepper = stepper
        self._level = level

    def __setitem__(self, alpha, value):
        super().__setitem__(alpha, np.asarray(value, dtype=float).copy())
        self._stepper._set_level(self._level, {alpha: value})


class CoupledStepper:
    """Leapfrog integrator for a set of coupled subdomain models (stepper.py:144-449).

    ``workers`` is accepted for signature compatibility; the GPU kernel is
    deterministic by construction, so results never depend on it.
    """

    def __init__(self, models: dict, dt: float, sources: Sequence[SourceTerm] = (), workers: int = 1,
                 device_coefficients=None, precision: str = "fp64"):
        """``device_coefficients``: optional (gammas, gamma_hats, scales) device
        addresses holding the chain stacks of all models in sorted(alpha) order
        (as ``build_models(..., device_out=...)`` writes them); the host arrays
        of the models are then not needed.

        ``precision``: "fp64" (U-form, the reference's arithmetic) or "fp32"
        (the W-form variant of SURVEY 8c.4: U_j = G_j W_j, Lanczos block-
        tridiagonal operator, half the bytes; within 1e-4 of fp64)."""
        if precision not in ("fp64", "fp32"):
            raise ConfigError("precision must be 'fp64' or 'fp32'")
        self.precision = precision
        if dt <= 0:
            raise ConfigError(f"time step must be positive, got {dt}")
        self.models = dict(models)
        self.order: list[Alpha] = sorted(self.models)
        self.dt = float(dt)
        self.sources = tuple(sources)
        self.workers = max(1, int(workers))
        for src in self.sources:
            if src.alpha not in self.models:
                raise ConfigError(f"source subdomain {src.alpha} has no model")
        self.index = {a: i for i, a in enumerate(self.order)}
        self._ifaces = self._pair_interfaces()
        self._ifaces_mass = None
        self.message_count = 0
        self.steps_done = 0
        self.time = 0.0
        self._baseline = 0.0
        self._initialized = False
        self._probe_key = None
        self._h = None
        self._devcoef = device_coefficients
        self._create()

    # -- setup -----------------------------------------------------------------

    def _pair_interfaces(self) -> list[Interface]:
        """Neighbour-table protocol checks of stepper.py:178-220 (bookkeeping only;
        the masses and the Gamma-hat_1 = I check run on the device)."""
        pairs = []
        for alpha in self.order:
            model = self.models[alpha]
            for face, beta in sorted(model.neighbors.items()):
                if beta not in self.models:
                    raise ProtocolError(f"subdomain {alpha} expects a neighbour {beta} across face {face} "
                                        "but no model was provided")
                other = self.models[beta]
                back = other.neighbors.get(opposite_face(face))
                if back != alpha:
                    raise ProtocolError(f"inconsistent neighbour tables: {alpha} face {face} points to "
                                        f"{beta}, whose opposite face points to {back}")
                if other.modes_per_face != model.modes_per_face:
                    raise ProtocolError(f"mode count mismatch across interface {alpha}|{beta}")
                if alpha < beta:
                    pairs.append(Interface(alpha, face, beta, opposite_face(face)))
        return pairs

    @property
    def interfaces(self) -> list[Interface]:
        """One Interface per shared face with its mass (stepper.py:178-220); the masses are
        computed on the device at create and copied back on first access."""
        if self._ifaces_mass is None:
            m = self._m
            masses = np.empty((max(1, len(self._ifaces)), m, m))
            cnt = C.c_int(0)
            eb = _lib.errbuf()
            _lib.check(self._lib.sfw_step_masses(self._h, C.byref(cnt), _lib.dptr(masses), eb, 1024), eb)
            self._ifaces_mass = [Interface(i.low, i.low_face, i.high, i.high_face, masses[q].copy())
                                 for q, i in enumerate(self._ifaces)]
        return self._ifaces_mass

    def _create(self):
        lib = _lib.load()
        ms = {self.models[a].modes_per_face for a in self.order}
        if len(ms) != 1:
            raise ConfigError("the GPU stepper needs one modes-per-face value for all subdomains")
        m = ms.pop()
        n = len(self.order)
        self._layers = np.array([self.models[a].layers for a in self.order], dtype=np.int32)
        self._sizes = self._layers.astype(np.int64) * 6 * m
        self._offs = np.concatenate([[0], np.cumsum(self._sizes)])
        nbr = np.full((n, 6), -1, dtype=np.int32)
        for i, a in enumerate(self.order):
            for f, b in self.models[a].neighbors.items():
                nbr[i, f] = self.index[b]
        if self._devcoef is None:
            gam = _f64(np.concatenate([np.asarray(self.models[a].gammas, float).reshape(-1) for a in self.order]))
            hat = _f64(np.concatenate([np.asarray(self.models[a].gamma_hats, float).reshape(-1)
                                       for a in self.order]))
            try:
                scl = _f64(np.concatenate([np.asarray(self.models[a].scales, float).reshape(-1)
                                           for a in self.order]))
            except (AttributeError, TypeError, ValueError):
                scl = None
            for i, a in enumerate(self.order):
                md = self.models[a]
                if np.shape(md.gammas) != (md.layers, 6 * m, 6 * m):
                    raise ConfigError(f"subdomain {a}: chain stacks must have shape (layers, 6m, 6m)")
            gptr, hptr, sptr = _lib.dptr(gam), _lib.dptr(hat), _lib.dptr(scl)
        else:
            gam = hat = scl = None
            gptr, hptr, sptr = (C.cast(C.c_void_p(int(x)), _lib.PD) if x else None for x in self._devcoef)
        src_sub = np.array([self.index[s.alpha] for s in self.sources], dtype=np.int32)
        for s in self.sources:
            if np.size(s.vector) != self.models[s.alpha].state_size:
                raise ConfigError(f"source vector for {s.alpha} has the wrong length")
        src_vec = _f64(np.concatenate([np.asarray(s.vector, float) for s in self.sources])) \
            if self.sources else np.zeros(1)
        self._src_norms = [float(np.linalg.norm(s.vector)) for s in self.sources]
        self._keep = (gam, hat, scl, nbr, src_sub, src_vec)
        d = _lib.StepDesc()
        d.n_sub = n
        d.m = m
        d.layers = _lib.iptr(self._layers)
        d.neighbors = _lib.iptr(np.ascontiguousarray(nbr.reshape(-1)))
        d.gammas = gptr
        d.gamma_hats = hptr
        d.scales = sptr
        d.coef_on_device = 0 if self._devcoef is None else 1
        d.dt = self.dt
        d.n_src = len(self.sources)
        d.src_sub = _lib.iptr(src_sub) if len(self.sources) else None
        d.src_vec = _lib.dptr(src_vec)
        d.n_probe = 0
        h = C.c_void_p()
        eb = _lib.errbuf()
        rc = lib.sfw_step_create(C.byref(d), C.byref(h), eb, 1024)
        _lib.check(rc, eb)
        self._h = h
        self._lib = lib
        self._m = m
        cnt = C.c_int(0)
        _lib.check(lib.sfw_step_masses(h, C.byref(cnt), None, eb, 1024), eb)
        if cnt.value != len(self._ifaces):
            raise ProtocolError(f"device paired {cnt.value} interfaces, host {len(self._ifaces)}")
        self._src_vec_u = src_vec
        self._probe_w_u = None
        if self.precision == "fp32":
            rc = lib.sfw_wform_setup(h, eb, 1024)
            _lib.check(rc, eb)
            self._wform_vectors()

    def _set_probes(self, probes: Sequence[Probe]):
        # the same Probe objects as the last upload (identity, O(n) in C): nothing to do
        prev = self._probe_key
        if prev is not None and len(prev) == len(probes) and all(map(operator.is_, probes, prev)):
            return
        key = tuple(probes)
        for p in probes:
            if p.alpha not in self.index:
                raise ConfigError(f"probe subdomain {p.alpha} has no model")
            if np.size(p.weights) != self.models[p.alpha].state_size:
                raise ConfigError(f"probe weights for {p.alpha} have the wrong length")
        sub = np.array([self.index[p.alpha] for p in probes], dtype=np.int32)
        w = _f64(np.concatenate([np.asarray(p.weights, float) for p in probes])) if probes else np.zeros(1)
        eb = _lib.errbuf()
        rc = self._lib.sfw_step_set_probes(self._h, len(probes), _lib.iptr(sub) if len(probes) else None,
                                           _lib.dptr(w), eb, 1024)
        _lib.check(rc, eb)
        self._probe_key = key
        self._probes = tuple(probes)
        self._probe_w_u = w
        if self.precision == "fp32":
            self._wform_vectors()

    def _wform_vectors(self):
        norms = np.zeros(max(1, len(self.sources)))
        eb = _lib.errbuf()
        rc = self._lib.sfw_wform_vectors(self._h, _lib.dptr(self._src_vec_u), _lib.dptr(self._probe_w_u),
                                         _lib.dptr(norms), eb, 1024)
        _lib.check(rc, eb)
        self._src_norms_w = norms[:len(self.sources)].tolist()

    # -- lifecycle -------------------------------------------------------------

    def close(self):
        if self._h is not None:
            if self.precision == "fp32":
                self._lib.sfw_wform_destroy(self._h)
            self._lib.sfw_step_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state marshalling -------------------------------------------------------

    def _concat(self, states: dict | None) -> np.ndarray | None:
        if not states:
            return None
        out = np.zeros(int(self._offs[-1]))
        for i, a in enumerate(self.order):
            if a in states:
                v = np.asarray(states[a], dtype=float)
                if v.size != self._sizes[i]:
                    raise ConfigError(f"state for {a} has the wrong length")
                out[self._offs[i]:self._offs[i + 1]] = v
        return out

    def _split(self, flat: np.ndarray) -> dict:
        return {a: flat[self._offs[i]:self._offs[i + 1]].copy() for i, a in enumerate(self.order)}

    def _state(self):
        uc = np.empty(int(self._offs[-1]))
        up = np.empty(int(self._offs[-1]))
        if self.precision == "fp32":
            eb = _lib.errbuf()
            _lib.check(self._lib.sfw_wform_state(self._h, _lib.dptr(uc), _lib.dptr(up), eb, 1024), eb)
        else:
            self._lib.sfw_step_get_state(self._h, _lib.dptr(uc), _lib.dptr(up))
        return uc, up

    @property
    def u_curr(self) -> dict:
        """Current state per subdomain (stepper.py:164).  A copy of the device state; item or
        attribute assignment writes back (the reference's dict is mutable)."""
        if not self._initialized:
            return {}
        return _StateView(self, 0, self._split(self._state()[0]))

    @u_curr.setter
    def u_curr(self, states: dict):
        self._set_level(0, states)

    @property
    def u_prev(self) -> dict:
        if not self._initialized:
            return {}
        return _StateView(self, 1, self._split(self._state()[1]))

    @u_prev.setter
    def u_prev(self, states: dict):
        self._set_level(1, states)

    def _set_level(self, level: int, states: dict):
        """Overwrite time level 0 (u_curr) or 1 (u_prev) for the subdomains in ``states``."""
        if self.precision != "fp64":
            raise ConfigError("assigning the state is defined for the fp64 U-form stepper")
        if not self._initialized:
            raise ProtocolError("stepper not initialized")
        flat = self._state()[level]
        for a, v in states.items():
            i = self.index[a]
            v = np.asarray(v, dtype=float).reshape(-1)
            if v.size != self._sizes[i]:
                raise ConfigError(f"state for {a} has the wrong length")
            flat[self._offs[i]:self._offs[i + 1]] = v
        flat = _f64(flat)
        eb = _lib.errbuf()
        rc = self._lib.sfw_step_set_state(self._h, _lib.dptr(flat) if level == 0 else None,
                                          _lib.dptr(flat) if level == 1 else None, eb, 1024)
        _lib.check(rc, eb)

    # -- physics -----------------------------------------------------------------

    def _acceleration(self, states: dict, count_messages: bool = False) -> dict:
        """Acceleration of a state (stepper.py:251-311), computed on the device."""
        if self.precision != "fp64":
            raise ConfigError("_acceleration is defined for the fp64 U-form stepper")
        flat = self._concat(states)
        if flat is None:
            flat = np.zeros(int(self._offs[-1]))
        out = np.empty_like(flat)
        eb = _lib.errbuf()
        rc = self._lib.sfw_step_accel(self._h, _lib.dptr(flat), None, _lib.dptr(out), eb, 1024)
        _lib.check(rc, eb)
        if count_messages:
            self.message_count += 2 * len(self._ifaces)
        return self._split(out)

    def _profiles(self, t_values) -> np.ndarray:
        tab = np.empty((len(self.sources), len(t_values)))
        for i, s in enumerate(self.sources):
            tab[i] = [float(v) for v in map(s.profile, t_values)]
        return np.ascontiguousarray(tab)

    def _profile_steps(self, k0: int, n: int) -> np.ndarray:
        """f_i(t_k), t_k = (k0 + k) dt for k < n: one row per source (stepper.py:313-321, 367)."""
        return profile_table([s.profile for s in self.sources], k0, n, self.dt, self._lib)

    def _limits(self, prof, norms_of_sources, n_steps):
        """Growth-detector thresholds of the next n_steps and the final baseline (stepper.py:379-389).

        The baseline gains dt*dt*|f_i(t_k)|*|src_i| per source and step, added in the
        reference's order (step-major, source-minor); np.add.accumulate is a sequential
        left-to-right sum, so the thresholds equal the reference's scalar loop bit for bit.
        """
        dt = self.dt
        if prof is None or not len(self.sources):
            base = np.full(n_steps, self._baseline)
        else:
            inc = (dt * dt * np.abs(prof.T)) * np.asarray(norms_of_sources, dtype=float)[None, :]  # (k, i)
            seq = np.concatenate([[self._baseline], inc.reshape(-1)])
            base = np.add.accumulate(seq)[len(self.sources)::len(self.sources)]
        return GROWTH_LIMIT * np.maximum(base, 1e-300), float(base[-1]) if n_steps else self._baseline

    # -- integration -------------------------------------------------------------

    def initialize(self, u0: dict | None = None, v0: dict | None = None, _probes: Sequence[Probe] = ()):
        """Two-level start, second-order accurate in dt (stepper.py:325-360)."""
        self._set_probes(_probes)
        u = self._concat(u0)
        v = self._concat(v0)
        prof = self._profiles([0.0]).reshape(-1) if self.sources else None
        row0 = np.empty(max(1, len(self._probes)))
        eb = _lib.errbuf()
        init = self._lib.sfw_wform_init if self.precision == "fp32" else self._lib.sfw_step_init
        rc = init(self._h, _lib.dptr(u), _lib.dptr(v), _lib.dptr(prof), _lib.dptr(row0), eb, 1024)
        _lib.check(rc, eb)
        self._row0 = row0[:len(self._probes)].copy()
        self.steps_done = 0
        self.time = 0.0
        self.message_count = 0
        dt = self.dt
        base = 0.0
        if u is not None or v is not None:  # from rest every term is 0.0
            for i, a in enumerate(self.order):
                uu = u[self._offs[i]:self._offs[i + 1]] if u is not None else np.zeros(int(self._sizes[i]))
                vv = v[self._offs[i]:self._offs[i + 1]] if v is not None else np.zeros(int(self._sizes[i]))
                base += float(np.linalg.norm(uu)) + dt * float(np.linalg.norm(vv))
        self._baseline = base
        self._initialized = True

    def _steps(self, n_steps: int, record_every: int, out: np.ndarray | None = None, check: bool = True):
        if not self._initialized:
            raise ProtocolError("stepper not initialized")
        dt = self.dt
        prof = self._profile_steps(self.steps_done, n_steps) if self.sources else None
        limits, base = self._limits(prof, self._src_norms, n_steps)
        if not check:
            limits = None
        n_rec = n_steps // record_every
        rows = out if out is not None else np.empty((max(1, n_rec), max(1, len(self._probes))))
        norms = np.empty(n_steps)
        bad = C.c_int(0)
        eb = _lib.errbuf()
        if self.precision == "fp32":
            # W-form: |W| against the same detector rule with W-form source norms, checked by the
            # library chunk by chunk (it stops launching at the first failing step)
            limits, base = self._limits(prof, self._src_norms_w, n_steps)
            if not check:
                limits = None
            ms = C.c_float(0.0)
            rc = self._lib.sfw_wform_run(self._h, n_steps, record_every, _lib.dptr(prof), _lib.dptr(limits),
                                         _lib.dptr(rows), _lib.dptr(norms), C.byref(bad), C.byref(ms), eb, 1024)
            self.last_kernel_ms = ms.value
        else:
            rc = self._lib.sfw_step_run(self._h, n_steps, record_every, _lib.dptr(prof), _lib.dptr(limits),
                                        _lib.dptr(rows), _lib.dptr(norms), C.byref(bad), eb, 1024)
        if rc == _lib.SFW_EINSTABLE:
            k = bad.value
            self.steps_done += k
            self.time = self.steps_done * dt
            raise InstabilityError(
                f"coupled stepping diverged at step {self.steps_done}: |U| = {norms[k - 1]:.3e} exceeds "
                f"{GROWTH_LIMIT:.0e} x reference {limits[k - 1] / GROWTH_LIMIT:.3e}")
        _lib.check(rc, eb)
        self._baseline = base
        self.message_count += n_steps * 2 * len(self._ifaces)
        start = self.steps_done
        self.steps_done += n_steps
        self.time = self.steps_done * dt
        steps = [start + k for k in range(record_every, n_steps + 1, record_every)]
        return steps, rows[:n_rec, :len(self._probes)]

    def advance(self):
        """One leapfrog step for all subdomains (stepper.py:362-389)."""
        self._steps(1, 1)

    def run(self, n_steps: int, probes: Sequence[Probe] = (), record_every: int = 1,
            u0: dict | None = None, v0: dict | None = None):
        """Step n_steps from rest (or given state), recording probes (stepper.py:391-412).

        Returns (times, samples): one row at t=0 and one after every
        ``record_every`` steps; one column per probe.  All steps run in one
        persistent kernel launch.
        """
        if record_every < 1:
            raise ConfigError("record_every must be at least 1")
        self.initialize(u0, v0, _probes=probes)
        n_rec = n_steps // record_every if n_steps > 0 else 0
        n_p = len(self._probes)
        # one output array: the library writes the probe rows straight into rows 1..n_rec
        out = np.empty((1 + n_rec, n_p)) if n_p else np.empty((1 + n_rec, 0))
        out[0] = self._row0
        start = self.steps_done
        if n_steps > 0:
            try:
                self._steps(n_steps, record_every, out=out[1:] if (n_p and n_rec) else None)
            except InstabilityError:
                # the persistent launch ran past the first failing step k; replay the k steps from
                # the same start (bitwise deterministic) so u_curr / u_prev / steps_done / time are
                # the reference's at the raise (stepper.py:379-389 stops at step k)
                k = self.steps_done - start
                self.initialize(u0, v0, _probes=probes)
                if k > 0:
                    self._steps(k, 1, check=False)
                raise
        times = np.concatenate([[0.0], (np.arange(record_every, n_steps + 1, record_every, dtype=np.float64)
                                        + float(start)) * self.dt]) if n_steps > 0 else np.zeros(1)
        return times, out

    # -- independent shots (BASELINE config 4) ------------------------------------

    SHOTS = 32

    def run_shots(self, n_steps: int, shots: Sequence[SourceTerm], probes: Sequence[Probe] = (),
                  record_every: int = 1, return_norms: bool = False):
        """Step up to 32 independent wavefields from rest in one launch.

        Shot q is exactly ``CoupledStepper(models, dt, sources=(shots[q],)).run(
        n_steps, probes, record_every)`` of the reference (SURVEY 8d config 4:
        32 separate runs); on the GPU all shots share one persistent kernel whose
        block products are (w x w)(w x 32) DMMA GEMMs.  Returns (times, rows) with
        rows[k, q, p] = probe p of shot q after the k-th recorded step (row 0 at t=0).
        """
        if record_every < 1:
            raise ConfigError("record_every must be at least 1")
        S = self.SHOTS
        if not 1 <= len(shots) <= S:
            raise ConfigError(f"run_shots takes 1..{S} shots")
        for sh in shots:
            if sh.alpha not in self.index:
                raise ConfigError(f"source subdomain {sh.alpha} has no model")
            if np.size(sh.vector) != self.models[sh.alpha].state_size:
                raise ConfigError(f"source vector for {sh.alpha} has the wrong length")
        self._set_probes(probes)
        eb = _lib.errbuf()
        prev = getattr(self, "_shots_key", None)
        if not (prev is not None and len(prev) == len(shots) and all(map(operator.is_, shots, prev))):
            sub = np.full(S, -1, dtype=np.int32)
            vecs = []
            for q, sh in enumerate(shots):
                sub[q] = self.index[sh.alpha]
                vecs.append(np.asarray(sh.vector, float))
            vec = _f64(np.concatenate(vecs))
            rc = self._lib.sfw_shots_setup(self._h, S, _lib.iptr(sub), _lib.dptr(vec), eb, 1024)
            _lib.check(rc, eb)
            self._shots_key = tuple(shots)
        dt = self.dt
        ns = len(shots)
        prof = np.zeros((S, n_steps))
        prof0 = np.zeros(S)
        prof[:ns] = profile_table([sh.profile for sh in shots], 0, n_steps, dt, self._lib)
        for q, sh in enumerate(shots):
            prof0[q] = float(sh.profile(0.0))
        n_rec = n_steps // record_every
        n_p = len(self._probes)
        out = np.empty((n_rec + 1, ns, n_p))
        out[0] = 0.0  # from rest: every probe reads 0 at t = 0
        # the library writes [record][shot][probe]: straight into out[1:] when all 32 shots are used
        direct = bool(ns == S and n_p and n_rec)
        rows = out[1:] if direct else np.zeros((max(n_rec, 1), S, max(n_p, 1)))
        norms = np.zeros((n_steps, S))
        ms = C.c_float(0.0)
        rc = self._lib.sfw_shots_run(self._h, n_steps, record_every, _lib.dptr(prof0), _lib.dptr(_f64(prof)),
                                     _lib.dptr(rows) if n_p else None, _lib.dptr(norms), C.byref(ms), eb, 1024)
        _lib.check(rc, eb)
        self.last_kernel_ms = ms.value
        if n_p and n_rec and not direct:
            out[1:] = rows[:n_rec, :ns, :n_p]
        # growth detector per shot (stepper.py:379-389), from rest: baseline_k = sum_{i<=k} dt^2 |f_i| |vec|,
        # accumulated left to right (np.cumsum is sequential), as the reference's scalar loop
        nv = np.array([float(np.linalg.norm(sh.vector)) for sh in shots])
        base = np.cumsum((dt * dt * np.abs(prof[:ns])) * nv[:, None], axis=1)
        bad = ~(norms[:, :ns].T <= GROWTH_LIMIT * np.maximum(base, 1e-300))
        if bad.any():
            q, k = min(zip(*np.nonzero(bad)), key=lambda qk: (qk[1], qk[0]))
            raise InstabilityError(f"shot {q}: coupled stepping diverged at step {k + 1}: |U| = {norms[k, q]:.3e}")
        self._initialized = False  # the single-wavefield state was not advanced
        times = np.array([0.0] + [k * dt for k in range(record_every, n_steps + 1, record_every)])
        if return_norms:
            return times, out, norms[:, :len(shots)]
        return times, out

    def shot_state(self, q: int):
        """(u_curr, u_prev) dicts of shot q after run_shots."""
        uc = np.empty(int(self._offs[-1]))
        up = np.empty(int(self._offs[-1]))
        self._lib.sfw_shots_state(self._h, int(q), _lib.dptr(uc), _lib.dptr(up))
        return self._split(uc), self._split(up)

    def shots_traffic(self):
        b, f, s = C.c_double(), C.c_double(), C.c_double()
        self._lib.sfw_shots_traffic(self._h, C.byref(b), C.byref(f), C.byref(s))
        return b.value, f.value, s.value

    # -- diagnostics -------------------------------------------------------------

    def energy(self) -> float:
        """Discrete invariant of the coupled leapfrog (stepper.py:419-449), on the device."""
        if not self._initialized:
            raise ProtocolError("stepper not initialized")
        if self.precision != "fp64":
            raise ConfigError("energy() is defined for the fp64 U-form stepper")
        e = C.c_double(0.0)
        eb = _lib.errbuf()
        rc = self._lib.sfw_step_energy(self._h, C.byref(e), eb, 1024)
        _lib.check(rc, eb)
        return e.value

    def traffic(self):
        """(algorithmic bytes, algorithmic flops, streamed bytes) per step."""
        b, f, s = C.c_double(), C.c_double(), C.c_double()
        self._lib.sfw_step_traffic(self._h, C.byref(b), C.byref(f), C.byref(s))
        return b.value, f.value, s.value


def profile_table(profiles, k0: int, n: int, dt: float, lib=None) -> np.ndarray:
    """[len(profiles), n] table of f(t_k), t_k = (k0 + k) * dt (the reference's int * float).

    Pulses from ``pulses.py`` carry ``sfw_pulse`` and are tabulated by the library with the
    same libm calls (bit-identical, tests/test_host_cpu.py); any other callable is evaluated
    per step in Python, as the reference does.
    """
    tab = np.empty((len(profiles), n))
    t_vals = None
    for i, f in enumerate(profiles):
        spec = getattr(f, "sfw_pulse", None)
        if spec is not None and n > 0:
            lib = lib or _lib.load()
            rc = lib.sfw_pulse_table(int(spec[0]), float(spec[1]), float(spec[2]), int(k0), float(dt), int(n),
                                     _lib.dptr(tab[i]))
            if rc == 0:
                continue
        if t_vals is None:
            t_vals = ((np.arange(n, dtype=np.float64) + float(k0)) * dt).tolist()
        tab[i] = [float(v) for v in map(f, t_vals)]
    return tab


def chain_operator(model: SubdomainModel) -> np.ndarray:
    """Dense isolated-subdomain operator (stepper.py:73-88) -- a test/diagnostic helper."""
    w, L = model.width, model.layers
    op = np.zeros((L * w, L * w))
    for j in range(L):
        blk = slice(j * w, (j + 1) * w)
        gp = model.gammas[j - 1] if j > 0 else np.zeros((w, w))
        op[blk, blk] = -model.gamma_hats[j] @ (model.gammas[j] + gp)
        if j > 0:
            op[blk, slice((j - 1) * w, j * w)] = model.gamma_hats[j] @ gp
        if j + 1 < L:
            op[blk, slice((j + 1) * w, (j + 2) * w)] = model.gamma_hats[j] @ model.gammas[j]
    return op


LAST_CFL: dict = {}


def cfl_estimate_coupled(models: dict, *, tol: float = POWER_TOL, max_iter: int = POWER_MAX_ITER,
                         seed: int = 0, device_coefficients=None) -> tuple[float, bool]:
    """Largest eigenvalue of the coupled second-derivative map (stepper.py:452-487).

    The start vector is drawn exactly as the reference does (numpy
    default_rng(seed), one standard-normal block per subdomain in sorted
    order); the iteration itself runs on the device.
    """
    with CoupledStepper(models, dt=1.0, device_coefficients=device_coefficients) as st:
        rng = np.random.default_rng(seed)
        x0 = np.concatenate([rng.standard_normal(models[a].state_size) for a in st.order])
        lam = C.c_double(0.0)
        conv = C.c_int(0)
        its = C.c_int(0)
        eb = _lib.errbuf()
        rc = st._lib.sfw_step_power(st._h, _lib.dptr(_f64(x0)), float(tol), int(max_iter), C.byref(lam),
                                    C.byref(conv), C.byref(its), eb, 1024)
        _lib.check(rc, eb)
    LAST_CFL.clear()
    LAST_CFL.update(iterations=its.value, converged=bool(conv.value))
    if not conv.value:
        log.warning("coupled CFL power iteration hit %d iterations", max_iter)
    return lam.value, bool(conv.value)


def stable_step_coupled(models: dict, **kw) -> tuple[float, float, bool]:
    """(dt_max, lambda_hat, converged) for the coupled system (stepper.py:490-495)."""
    lam, converged = cfl_estimate_coupled(models, **kw)
    if lam <= 0:
        raise NumericalError("coupled operator has no negative spectrum")
    return 2.0 / np.sqrt(lam), lam, converged




DT_SAFETY = CFL_SAFETY  # sim.py:63


def resolve_dt(dt, dt_max_coupled: float, converged: bool, dt_max_fine: float) -> float:
    """The reference's time-step policy (sim.py:444-463 ``_resolve_dt``) over a dt spec.

    ``dt``: "auto" (0.9 x the coupled limit, or 0.9 x the fine-grid limit when the coupled power
    iteration did not converge), "fine" (0.9 x the fine-grid limit) or a number, which must not
    exceed 0.9 x the coupled limit (relative slack 1e-12) -- ConfigError("...", "time.dt") otherwise.
    ``dt_max_coupled`` = 2/sqrt(lambda) of ``cfl_estimate_coupled`` (GPU), ``dt_max_fine`` =
    ``fdtd.stability_limit`` of the global operator (GPU).
    """
    if dt == "auto":
        if converged:
            return DT_SAFETY * dt_max_coupled
        log.warning("coupled stability estimate did not converge; falling back to the fine-grid step")
        return DT_SAFETY * dt_max_fine
    if dt == "fine":
        return DT_SAFETY * dt_max_fine
    val = float(dt)
    limit = DT_SAFETY * dt_max_coupled
    if val > limit * (1.0 + 1e-12):
        raise ConfigError(f"requested dt {val:.6e} exceeds the stable limit {limit:.6e}", "time.dt")
    return val


def _resolve_dt(config, dt_max_coupled: float, converged: bool, dt_max_fine: float) -> float:
    """Reference-shaped form (sim.py:444): ``config`` is any object with a ``dt`` attribute."""
    return resolve_dt(config.dt, dt_max_coupled, converged, dt_max_fine)


__all__ = [
    "CFL_SAFETY", "CoupledStepper", "DT_SAFETY", "FaceMessage", "Interface", "Probe", "SourceTerm", "chain_operator",
    "cfl_estimate_coupled", "make_probe", "project_source", "resolve_dt", "stable_step_coupled",
]
