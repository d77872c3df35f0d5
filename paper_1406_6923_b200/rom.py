"""Off-line ROM data model (mirror of reference rom.py:319-356 SubdomainModel).

The batched sm_100a build pipeline lives in ``romgpu.py`` / ``csrc/sfw_rom.cu``;
``build_subdomain_model`` keeps the reference signature (rom.py:359-364).
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


class _RomDesc(_C.Structure):
    _fields_ = [("n_sub", _C.c_int), ("p", _C.c_int * 3), ("h", _C.c_double * 3), ("m", _C.c_int),
                ("n", _C.c_int), ("shift", _C.c_double), ("c", _lib.PD), ("nbr_mask", _lib.PI),
                ("n_rows", _C.c_int), ("row_sub", _lib.PI), ("row_node", _lib.PI), ("full_basis", _C.c_int),
                ("out_on_device", _C.c_int), ("batch", _C.c_int)]


class _RomOut(_C.Structure):
    _fields_ = [("layers", _lib.PI), ("flags", _lib.PI), ("status", _lib.PI), ("gammas", _lib.PD),
                ("gamma_hats", _lib.PD), ("scales", _lib.PD), ("tdiag", _lib.PD), ("toff", _lib.PD),
                ("basis_rows", _lib.PD), ("basis", _lib.PD), ("stats", _lib.PD)]


_lib.SIGNATURES["sfw_rom_build"] = (_C.c_int, [_C.POINTER(_RomDesc), _C.POINTER(_RomOut), _C.c_char_p, _C.c_int])

LAST_BUILD_STATS: dict = {}


def _mask(neighbors) -> int:
    return sum(1 << f for f in neighbors)


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
    if not hasattr(lib.sfw_rom_build, "_typed"):
        fn = lib.sfw_rom_build
        fn.restype, fn.argtypes = _lib.SIGNATURES["sfw_rom_build"]
        fn._typed = True
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
    d = _RomDesc()
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
    o = _RomOut()
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
