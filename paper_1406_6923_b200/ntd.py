"""Reduced boundary transfer maps on the GPU (mirror of reference ntd.py, reduced forms).

For a symmetric negative semidefinite operator A and orthonormal face inputs
F, the Neumann-to-Dirichlet map at angular frequency w is
``M(w) = F* (A + w^2 I)^-1 F``.  The reference evaluates it in four forms and
cross-checks them (ntd.py, sim.verify_subdomain, acceptance criterion 1).
Here the two forms a GPU-built model carries -- the block-tridiagonal Lanczos
form (``ntd_tridiag``, ntd.py:101-146) and the S-fraction chain
(``ntd_chain``, ntd.py:149-185) -- run batched on the device, one CTA per
(model, frequency) (``sfw_ntd_batch``, csrc/sfw_ntd.cu).  ``frequency_band`` /
``nudge_off_poles`` are the reference's host bookkeeping.

Not here: ``ntd_full`` / ``band_error`` (a sparse indefinite direct solve of
the N x N operator per frequency) and ``ntd_reduced`` (needs the projected
pair, which the GPU build does not keep).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError

RESONANCE_RTOL = 1e-6
POLE_RTOL = 1e-8


def frequency_band(omega_min: float, omega_max: float, count: int = 20) -> np.ndarray:
    """Log-spaced angular frequencies over [omega_min, omega_max] (ntd.py:30-38)."""
    if not (0 < omega_min < omega_max):
        raise ConfigError(f"need 0 < omega_min < omega_max, got [{omega_min}, {omega_max}]")
    if count < 1:
        raise ConfigError(f"need at least one frequency, got {count}")
    return np.geomspace(omega_min, omega_max, count)


def nudge_off_poles(omegas: np.ndarray, poles: np.ndarray) -> np.ndarray:
    """Move frequencies within POLE_RTOL of a pole up until clear (ntd.py:41-59)."""
    out = np.array(omegas, dtype=float)
    if poles.size == 0:
        return out
    for i, w in enumerate(out):
        step = 10.0 * POLE_RTOL * max(w, 1.0)
        for _ in range(100):
            if np.min(np.abs(poles - out[i])) > POLE_RTOL * max(out[i], 1.0):
                break
            out[i] += step
    return out


def _batch(form: int, a_stack, b_stack, e_stack, item_model, omegas):
    a_stack = np.ascontiguousarray(a_stack, dtype=np.float64)
    n_models, layers, w, _ = a_stack.shape
    b_stack = np.ascontiguousarray(b_stack, dtype=np.float64)
    e_stack = None if e_stack is None else np.ascontiguousarray(e_stack, dtype=np.float64)
    im = np.ascontiguousarray(item_model, dtype=np.int32)
    om = np.ascontiguousarray(omegas, dtype=np.float64)
    out = np.empty((im.size, w, w))
    status = np.zeros(im.size, dtype=np.int32)
    lib = _lib.load()
    eb = _lib.errbuf()
    b_ptr = _lib.dptr(b_stack) if b_stack.size else _lib.dptr(np.zeros(1))
    _lib.check(lib.sfw_ntd_batch(form, n_models, layers, w, _lib.dptr(a_stack), b_ptr, _lib.dptr(e_stack), im.size,
                                 _lib.iptr(im), _lib.dptr(om), _lib.dptr(out), _lib.iptr(status), eb, 1024), eb,
               "sfw_ntd_batch")
    bad = np.nonzero(status)[0]
    if bad.size:
        raise NumericalError(f"{'tridiagonal' if form == 0 else 'chain'} transfer map is singular at omega = "
                             f"{om[bad[0]]:.6e}")
    return out


def ntd_tridiag(diag_blocks, off_blocks, entry_block, omega: float) -> np.ndarray:
    """Transfer map from the block tridiagonal form (ntd.py:101-146): Schur chain, assembled fallback."""
    d = np.asarray(diag_blocks, dtype=float)[None]
    b = np.asarray(off_blocks, dtype=float).reshape((1, max(d.shape[1] - 1, 0)) + d.shape[2:])
    e = np.asarray(entry_block, dtype=float)[None]
    return _batch(0, d, b, e, [0], [float(omega)])[0]


def ntd_chain(gammas, gamma_hats, omega: float) -> np.ndarray:
    """Transfer map from the chain coefficients (ntd.py:149-185)."""
    g = np.asarray(gammas, dtype=float)[None]
    h = np.asarray(gamma_hats, dtype=float)[None]
    return _batch(1, g, h, None, [0], [float(omega)])[0]


def ntd_batch(models, omegas, form: str = "chain") -> np.ndarray:
    """Maps of many models at many frequencies: array [len(models), len(omegas), w, w].

    ``form="chain"`` uses ``gammas`` / ``gamma_hats``; ``form="tridiag"`` the
    Lanczos blocks ``tdiag`` / ``toff`` and ``entry`` (identity when a model
    has no ``entry``: the GPU build's gauge makes the entry block I to ~1e-14).
    All models must share the layer count and width.
    """
    models = list(models)
    omegas = np.asarray(omegas, dtype=float).ravel()
    if not models or omegas.size == 0:
        raise ConfigError("ntd_batch needs at least one model and one frequency")
    nm, nw = len(models), omegas.size
    item_model = np.repeat(np.arange(nm), nw)
    item_omega = np.tile(omegas, nm)
    if form == "chain":
        a = np.stack([m.gammas for m in models])
        b = np.stack([m.gamma_hats for m in models])
        out = _batch(1, a, b, None, item_model, item_omega)
    elif form == "tridiag":
        a = np.stack([m.tdiag for m in models])
        b = np.stack([m.toff for m in models])
        w = a.shape[-1]
        e = np.stack([getattr(m, "entry", None) if getattr(m, "entry", None) is not None else np.eye(w)
                      for m in models])
        out = _batch(0, a, b, e, item_model, item_omega)
    else:
        raise ConfigError("form must be 'chain' or 'tridiag'")
    return out.reshape(nm, nw, *out.shape[1:])
