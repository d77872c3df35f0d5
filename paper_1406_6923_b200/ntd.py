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

The explicit-operator forms -- ``ntd_full`` (the sparse N x N subdomain
operator, ntd.py:62-98), ``ntd_reduced`` (the dense projected pair,
ntd.py:101-115) and ``band_error`` (ntd.py:188-202) -- run on the device too
(``sfw_ntd_operator``, csrc/sfw_ntdfull.cu): band LU with partial pivoting of
A + w^2 I, one CTA per frequency, with the reference's residual-based
resonance test.  The reference factors with SuperLU, so these agree with it to
the conditioning of the shifted operator rather than bit for bit.
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


def _csr(matrix):
    """Host CSR (int32 indices) of a scipy sparse matrix or a dense array."""
    from scipy import sparse
    m = matrix.tocsr() if sparse.issparse(matrix) else sparse.csr_matrix(np.asarray(matrix, dtype=float))
    m.sort_indices()
    return (np.ascontiguousarray(m.indptr, dtype=np.int32), np.ascontiguousarray(m.indices, dtype=np.int32),
            np.ascontiguousarray(m.data, dtype=np.float64), m.shape[0])


def _operator_maps(matrix, f, omegas):
    rp, ci, val, n = _csr(matrix)
    f = np.ascontiguousarray(np.asarray(f, dtype=float).reshape(n, -1))
    om = np.ascontiguousarray(np.asarray(omegas, dtype=float).ravel())
    w = f.shape[1]
    out = np.empty((om.size, w, w))
    resid = np.empty(om.size)
    status = np.zeros(om.size, dtype=np.int32)
    lib = _lib.load()
    eb = _lib.errbuf()
    _lib.check(lib.sfw_ntd_operator(n, _lib.iptr(rp), _lib.iptr(ci), _lib.dptr(val), w, _lib.dptr(f), om.size,
                                    _lib.dptr(om), _lib.dptr(out), _lib.dptr(resid), _lib.iptr(status), eb, 1024),
               eb, "sfw_ntd_operator")
    return out, resid, status, om


def ntd_full_band(matrix, f: np.ndarray, omegas) -> np.ndarray:
    """ntd_full at many frequencies in one device call: array [len(omegas), w, w]."""
    out, resid, status, om = _operator_maps(matrix, f, omegas)
    for k, w in enumerate(om):
        if status[k]:
            raise NumericalError(f"transfer map solve failed at omega = {w:.6e}: matrix is exactly singular")
        if not resid[k] <= RESONANCE_RTOL:
            raise NumericalError(f"omega = {w:.6e} is resonant (relative residual {resid[k]:.2e}); "
                                 "move the frequency off the operator spectrum")
    return out


def ntd_full(matrix, f: np.ndarray, omega: float) -> np.ndarray:
    """F* (A + w^2 I)^-1 F of the full operator (ntd.py:62-98)."""
    return ntd_full_band(matrix, f, [float(omega)])[0]


def ntd_reduced(a_tilde: np.ndarray, f_tilde: np.ndarray, omega: float) -> np.ndarray:
    """Transfer map of the Galerkin-projected pair (ntd.py:101-115)."""
    out, _, status, _ = _operator_maps(np.asarray(a_tilde, dtype=float), f_tilde, [float(omega)])
    if status[0]:
        raise NumericalError(f"reduced transfer map is singular at omega = {float(omega):.6e}")
    return out[0]


def band_error(matrix, f: np.ndarray, a_tilde: np.ndarray, f_tilde: np.ndarray, omegas) -> float:
    """Max relative deviation of the projected map from the full map (ntd.py:188-202)."""
    om = np.asarray(omegas, dtype=float).ravel()
    exact = ntd_full_band(matrix, f, om)
    approx, _, status, _ = _operator_maps(np.asarray(a_tilde, dtype=float), f_tilde, om)
    worst = 0.0
    for k, w in enumerate(om):
        if status[k]:
            raise NumericalError(f"reduced transfer map is singular at omega = {w:.6e}")
        denom = max(np.linalg.norm(exact[k]), 1e-300)
        worst = max(worst, float(np.linalg.norm(approx[k] - exact[k]) / denom))
    return worst


def subdomain_inputs(op, modes: int) -> np.ndarray:
    """(N, 6 modes) face-input matrix F of a subdomain (rom.py:74-86), built on the device by the
    ROM pipeline's face-basis kernel: orthonormal tensor cosine modes on each owned face window."""
    px, py, pz = (int(s) for s in op.shape)
    n = px * py * pz
    out = np.empty((6 * modes, n))
    mask = sum(1 << f for f in op.neighbors)
    lib = _lib.load()
    eb = _lib.errbuf()
    _lib.check(lib.sfw_face_inputs(px, py, pz, int(modes), int(mask), _lib.dptr(out), eb, 1024), eb,
               "sfw_face_inputs")
    return np.ascontiguousarray(out.T)


def _tridiag_pair(model):
    """(T, [E; 0]): the block-Lanczos pair of a GPU-built model, assembled as ntd.py:130-139 does.
    Its transfer map is the projected pair's (V^T A V, V^T F) up to the orthogonal Q."""
    d = np.asarray(model.tdiag, dtype=float)
    b = np.asarray(model.toff, dtype=float)
    L, w = d.shape[0], d.shape[1]
    t = np.zeros((L * w, L * w))
    for j in range(L):
        blk = slice(j * w, (j + 1) * w)
        t[blk, blk] = d[j]
        if j + 1 < L:
            nxt = slice((j + 1) * w, (j + 2) * w)
            t[nxt, blk] = b[j]
            t[blk, nxt] = b[j].T
    e = getattr(model, "entry", None)
    ft = np.zeros((L * w, w))
    ft[:w] = np.eye(w) if e is None else e
    return t, ft


def verify_subdomain(op, modes_per_face: int, shift: float, omegas, n_max: int = 5) -> dict:
    """Transfer-map accuracy of one subdomain's reduction, depth by depth (sim.py:703-768).

    ``op``: a subdomain operator with its host matrix (``grid.assemble_subdomain_operator(...,
    with_matrix=True)``); ``omegas``: the verification band (the reference's ``source_band``).
    For n = 1..n_max the GPU-built model's block-Lanczos pair is compared with the full
    operator over the band (``band_error``); at n_max its reduced, tridiagonal and chain maps
    are cross-checked at the quarter of the band farthest from the reduced spectrum.  Every
    solve runs on the device; the pole ranking of the probe frequencies is host bookkeeping.
    """
    from .rom import build_models
    if getattr(op, "matrix", None) is None:
        raise ConfigError("verify_subdomain needs the operator matrix (assemble_subdomain_operator(..., "
                          "with_matrix=True))")
    om = np.asarray(omegas, dtype=float).ravel()
    f = subdomain_inputs(op, modes_per_face)
    exact = ntd_full_band(op.matrix, f, om)
    rows = []
    model = None
    for n in range(1, n_max + 1):
        model = build_models([op], modes_per_face, n, shift)[op.alpha]
        t, ft = _tridiag_pair(model)
        approx, _, status, _ = _operator_maps(t, ft, om)
        worst = 0.0
        for k, w in enumerate(om):
            if status[k]:
                raise NumericalError(f"reduced transfer map is singular at omega = {w:.6e}")
            denom = max(np.linalg.norm(exact[k]), 1e-300)
            worst = max(worst, float(np.linalg.norm(approx[k] - exact[k]) / denom))
        rows.append((n, worst))
    t, ft = _tridiag_pair(model)
    poles = np.sqrt(np.maximum(-np.linalg.eigvalsh(t), 0.0))
    probe = np.array(sorted(om, key=lambda w: -float(np.min(np.abs(poles - w)) / w))[:max(1, om.size // 4)])
    base, _, status, _ = _operator_maps(t, ft, probe)
    if status.any():
        raise NumericalError(f"reduced transfer map is singular at omega = {probe[np.nonzero(status)[0][0]]:.6e}")
    tri = ntd_batch([model], probe, "tridiag")[0]
    chn = ntd_batch([model], probe, "chain")[0]
    agreement = 0.0
    for k in range(probe.size):
        scale = max(float(np.linalg.norm(base[k])), 1e-300)
        agreement = max(agreement, float(np.linalg.norm(tri[k] - base[k])) / scale,
                        float(np.linalg.norm(chn[k] - base[k])) / scale)
    return {"alpha": op.alpha, "omegas": om, "rows": rows, "agreement": agreement,
            "truncated": bool(getattr(model, "truncated", False))}
