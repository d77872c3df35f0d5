"""Off-line ROM stage: data model (reference rom.py:319-356 SubdomainModel), the batched
sm_100a build (``build_models`` -> ``sfw_rom_build`` in csrc/sfw_rom.cu) behind the reference
signature ``build_subdomain_model`` (rom.py:359-364), and the node/chain maps ``project_state``
/ ``state_to_nodes`` (rom.py:437-459, ``sfw_project_state`` / ``sfw_state_to_nodes``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NumericalError


@dataclass
class SubdomainModel:
    """Everything the online stage needs for one subdomain (rom.py:319-356).

    The chain stacks have shape (layers, 6m, 6m); ``basis`` is the node-space
    image V Q of the reduction basis (optional: only source / receiver
    subdomains need it, as in sim.load_models, sim.py:359-398).  ``tdiag`` /
    ``toff`` keep the block-Lanczos blocks (A_j, B_j), the best-conditioned
    parity targets.
    """

    alpha: tuple
    lo: tuple
    shape: tuple
    spacing: tuple
    modes_per_face: int
    layers: int
    shift: float
    neighbors: dict
    face_indices: tuple
    gammas: np.ndarray
    gamma_hats: np.ndarray
    scales: np.ndarray
    basis: np.ndarray | None
    c: np.ndarray
    mu: np.ndarray
    deflated: bool = False
    truncated: bool = False
    tdiag: np.ndarray | None = None
    toff: np.ndarray | None = None
    basis_rows: dict | None = None

    @property
    def width(self) -> int:
        return 6 * self.modes_per_face

    def face_slice(self, face: int) -> slice:
        m = self.modes_per_face
        return slice(face * m, (face + 1) * m)

    @property
    def state_size(self) -> int:
        return self.layers * self.width


def basis_row(model, row: int) -> np.ndarray:
    """Row ``row`` of the node-space basis V Q: from the full basis, or from the
    rows a batched build materialised (``build_models(rows=...)``)."""
    b = getattr(model, "basis", None)
    if b is not None:
        return np.asarray(b[row])
    rows = getattr(model, "basis_rows", None)
    if rows and int(row) in rows:
        return rows[int(row)]
    raise NumericalError("model was loaded without its node-space basis")


def require_basis(model) -> np.ndarray:
    if getattr(model, "basis", None) is None:
        raise NumericalError("model was loaded without its node-space basis")
    return model.basis


# ---------------------------------------------------------------------------
# batched sm_100a build (csrc/sfw_rom.cu) behind the reference signature

import ctypes as _C  # noqa: E402
import math as _math  # noqa: E402

from . import _lib  # noqa: E402
from .errors import ConfigError  # noqa: E402


LAST_BUILD_STATS: dict = {}


def _mask(neighbors) -> int:
    return sum(1 << f for f in neighbors)


def check_operators(ops, shape, spacing, c, masks, tol: float = 1e-10):
    """The GPU build never reads ``op.matrix``: it rebuilds the operator from (c, mu, h, neighbours)
    as the stencil A = -C S C of grid.py:415-458.  When an operator carries an explicit matrix (a
    reference ``SubdomainOperator`` always does), apply both to one seeded random vector -- the
    stencil on the device (``sfw_subdomain_apply``) -- and refuse operators that differ, instead
    of silently building a model of another operator."""
    idx = [i for i, op in enumerate(ops) if getattr(op, "matrix", None) is not None]
    if not idx:
        return
    lib = _lib.load()
    N = int(np.prod(shape))
    x = np.random.default_rng(1406).standard_normal(N)
    p = np.array(shape, dtype=np.int32)
    h = np.array(spacing, dtype=np.float64)
    for s0 in range(0, len(idx), 512):
        sel = idx[s0:s0 + 512]
        X = np.ascontiguousarray(np.broadcast_to(x, (len(sel), N)))
        Y = np.empty((len(sel), N))
        eb = _lib.errbuf()
        rc = lib.sfw_subdomain_apply(len(sel), _lib.iptr(p), _lib.dptr(h), _lib.dptr(np.ascontiguousarray(c[sel])),
                                     _lib.iptr(np.ascontiguousarray(masks[sel])), 1, _lib.dptr(X), _lib.dptr(Y),
                                     eb, 1024)
        _lib.check(rc, eb, "operator check")
        for k, i in enumerate(sel):
            mat = ops[i].matrix
            if getattr(mat, "shape", None) != (N, N):
                raise ConfigError(f"subdomain {ops[i].alpha}: operator matrix has shape {getattr(mat, 'shape', None)}, "
                                  f"expected {(N, N)}")
            want = np.asarray(mat @ x, dtype=np.float64).reshape(-1)
            err = float(np.linalg.norm(Y[k] - want)) / max(float(np.linalg.norm(want)), 1e-300)
            if not err <= tol:
                raise ConfigError(f"subdomain {ops[i].alpha}: op.matrix is not the finite-volume operator of its "
                                  f"(c, mu, spacing, neighbours) (relative mismatch {err:.2e}); the GPU build "
                                  "assembles that operator itself and cannot take an arbitrary matrix")


def build_models(ops, modes_per_face: int, n: int, shift: float, basis=None, rows=None, batch: int = 0,
                 device_out=None) -> dict:
    """Build the S-fraction models of many subdomains in one batched GPU pipeline.

    ``ops``: sequence of objects with ``alpha, lo, shape, spacing, c, mu,
    neighbors`` (reference ``SubdomainOperator`` or grid.SubdomainOperator).
    ``basis``: "all" (full V Q per model, as the reference stores it), None, or
    a set of alphas that need it (sim.load_models need_basis, sim.py:359-398).
    ``rows``: optional {alpha: [local rows]} -> ``model.basis_rows[row]``
    (K-vectors of V Q) without materialising the N x K basis.
    ``device_out``: optional (gammas, gamma_hats, scales) device pointers
    (int addresses) receiving the chain stacks directly in HBM.
    """
    lib = _lib.load()
    ops = list(ops)
    if not ops:
        return {}
    shape = tuple(ops[0].shape)
    spacing = tuple(ops[0].spacing)
    for op in ops:
        if tuple(op.shape) != shape or tuple(op.spacing) != spacing:
            raise ConfigError("a batched build needs one subdomain shape and spacing")
    k = _math.isqrt(modes_per_face)
    if k * k != modes_per_face:
        raise ConfigError(f"modes per face must be a perfect square, got {modes_per_face}")
    from .grid import face_window
    for op in ops:
        for f in range(6):
            na, nb = face_window(shape, f, op.neighbors).plane_shape
            if k > na or k > nb:
                raise ConfigError(f"{modes_per_face} modes need {k} per axis but the face window is {na}x{nb}")
    w = 6 * modes_per_face
    L = n + 1
    K = L * w
    N = int(np.prod(shape))
    ns = len(ops)
    c = np.ascontiguousarray(np.stack([np.asarray(op.c, dtype=np.float64).reshape(-1) for op in ops]))
    masks = np.array([_mask(op.neighbors) for op in ops], dtype=np.int32)
    check_operators(ops, shape, spacing, c, masks)
    want_basis = set()
    if basis == "all":
        want_basis = {op.alpha for op in ops}
    elif basis:
        want_basis = set(basis)
    full = bool(want_basis)
    row_sub, row_node = [], []
    index = {op.alpha: i for i, op in enumerate(ops)}
    for a, rr in (rows or {}).items():
        for r in rr:
            row_sub.append(index[a])
            row_node.append(int(r))
    row_sub = np.array(row_sub or [0], dtype=np.int32)
    row_node = np.array(row_node or [0], dtype=np.int32)
    n_rows = len(row_sub) if rows else 0
    d = _lib.RomDesc()
    d.n_sub = ns
    d.p[:] = shape
    d.h[:] = spacing
    d.m = modes_per_face
    d.n = n
    d.shift = float(shift)
    d.c = _lib.dptr(c)
    d.nbr_mask = _lib.iptr(masks)
    d.n_rows = n_rows
    d.row_sub = _lib.iptr(row_sub)
    d.row_node = _lib.iptr(row_node)
    d.full_basis = 1 if full else 0
    d.batch = int(batch)
    layers = np.zeros(ns, dtype=np.int32)
    flags = np.zeros(ns, dtype=np.int32)
    status = np.zeros(ns, dtype=np.int32)
    stats = np.zeros(16)
    o = _lib.RomOut()
    o.layers = _lib.iptr(layers)
    o.flags = _lib.iptr(flags)
    o.status = _lib.iptr(status)
    if device_out is None:
        gam = np.empty((ns, L, w, w))
        hat = np.empty((ns, L, w, w))
        scl = np.empty((ns, L, w, w))
        o.gammas, o.gamma_hats, o.scales = _lib.dptr(gam), _lib.dptr(hat), _lib.dptr(scl)
        d.out_on_device = 0
    else:
        gam = hat = scl = None
        o.gammas = _C.cast(_C.c_void_p(device_out[0]), _lib.PD)
        o.gamma_hats = _C.cast(_C.c_void_p(device_out[1]), _lib.PD)
        o.scales = _C.cast(_C.c_void_p(device_out[2]), _lib.PD)
        d.out_on_device = 1
    tdiag = np.empty((ns, L, w, w))
    toff = np.empty((ns, max(L - 1, 1), w, w))
    o.tdiag = _lib.dptr(tdiag)
    o.toff = _lib.dptr(toff)
    brows = np.empty((max(n_rows, 1), K))
    o.basis_rows = _lib.dptr(brows)
    bas = np.empty((ns, K, N)) if full else None
    o.basis = _lib.dptr(bas) if full else None
    o.stats = _lib.dptr(stats)
    eb = _lib.errbuf()
    rc = lib.sfw_rom_build(_C.byref(d), _C.byref(o), eb, 1024)
    _lib.check(rc, eb)
    LAST_BUILD_STATS.clear()
    LAST_BUILD_STATS.update(dict(zip(["solve_s", "orth_s", "project_s", "lanczos_s", "sfraction_s",
                                      "max_pcg_iters", "batch", "wall_s"], stats[:8].tolist())))
    out = {}
    rows_by = {}
    t = 0
    for a, rr in (rows or {}).items():
        for r in rr:
            rows_by.setdefault(a, {})[int(r)] = brows[t]
            t += 1
    for i, op in enumerate(ops):
        a = op.alpha
        Li = int(layers[i])
        md = SubdomainModel(
            alpha=a, lo=tuple(op.lo), shape=shape, spacing=spacing, modes_per_face=modes_per_face,
            layers=Li, shift=float(shift), neighbors=dict(op.neighbors),
            face_indices=tuple(getattr(op, "face_nodes")[f].indices for f in range(6))
            if hasattr(op, "face_nodes") else (),
            gammas=gam[i][:Li] if gam is not None else None, gamma_hats=hat[i][:Li] if hat is not None else None,
            scales=scl[i][:Li] if scl is not None else None,
            basis=np.ascontiguousarray(bas[i][:Li * w].T) if (full and a in want_basis) else None,
            c=np.asarray(op.c, dtype=float).reshape(-1), mu=np.asarray(op.mu, dtype=float).reshape(-1),
            deflated=bool(flags[i] & 1), truncated=bool(flags[i] & 2), tdiag=tdiag[i][:Li],
            toff=toff[i][:Li - 1])
        if a in rows_by:
            md.basis_rows = {r: v[:Li * w].copy() for r, v in rows_by[a].items()}
        out[a] = md
    return out


def build_subdomain_model(op, modes_per_face: int, n: int, shift: float) -> SubdomainModel:
    """Run the full offline pipeline for one subdomain operator (rom.py:359-434), on the GPU."""
    return build_models([op], modes_per_face, n, shift, basis="all")[op.alpha]


def _state_map(fn, model, vec, n_in, n_out, what):
    basis = require_basis(model)
    lib = _lib.load()
    L, w = model.layers, model.width
    N = int(basis.shape[0])
    x = np.ascontiguousarray(np.asarray(vec, dtype=np.float64).reshape(-1))
    if x.size != (N if n_in == "N" else L * w):
        raise ConfigError(f"{what}: input has length {x.size}")
    out = np.empty(N if n_out == "N" else L * w)
    eb = _lib.errbuf()
    rc = getattr(lib, fn)(N, L, w, _lib.dptr(np.ascontiguousarray(basis, dtype=np.float64)),
                          _lib.dptr(np.ascontiguousarray(model.scales, dtype=np.float64)), _lib.dptr(x),
                          _lib.dptr(out), eb, 1024)
    _lib.check(rc, eb, what)
    return out


def project_state(model: SubdomainModel, w: np.ndarray) -> np.ndarray:
    """Map a node-space field (symmetrized variable) to chain layers (rom.py:437-447), on the GPU."""
    return _state_map("sfw_project_state", model, w, "N", "K", "project_state")


def state_to_nodes(model: SubdomainModel, u: np.ndarray) -> np.ndarray:
    """Inverse of project_state on the reduction subspace (rom.py:450-459), on the GPU."""
    return _state_map("sfw_state_to_nodes", model, u, "K", "N", "state_to_nodes")
