"""Host-side geometry: tiling, ownership and face windows (mirror of reference grid.py).

Only bookkeeping lives here (index sets, multiplicities, the sampled sound
speed); the fine-grid operator A = D K D of reference grid.py:326-458 is never
assembled on the host -- the sm_100a ROM build applies it as a stencil from
(c, per-axis multiplicities, h).  ``assemble_subdomain_operator`` therefore
returns a ``SubdomainOperator`` whose ``matrix`` is None unless requested.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError

FACE_AXIS = (0, 0, 1, 1, 2, 2)
FACE_SIDE = (0, 1, 0, 1, 0, 1)


def opposite_face(face: int) -> int:
    return face ^ 1


@dataclass(frozen=True)
class DomainSpec:
    """Global box and its tiling (grid.py:45-85); adjacent subdomains share a node layer."""

    extents: tuple
    subdomain_counts: tuple
    nodes_per_subdomain: tuple
    outer_bc: str = "reflecting"

    def __post_init__(self):
        if len(self.extents) != 3 or any(e <= 0 for e in self.extents):
            raise ConfigError("extents must be three positive numbers", "domain.extents")
        if len(self.subdomain_counts) != 3 or any(c < 1 for c in self.subdomain_counts):
            raise ConfigError("subdomain counts must be >= 1", "domain.subdomains")
        if len(self.nodes_per_subdomain) != 3 or any(p < 4 for p in self.nodes_per_subdomain):
            raise ConfigError("nodes per subdomain must be >= 4", "domain.nodes_per_subdomain")
        if self.outer_bc not in ("reflecting", "sponge"):
            raise ConfigError("outer_bc must be 'reflecting' or 'sponge'", "domain.outer_bc")

    @property
    def global_shape(self) -> tuple:
        return tuple(c * (p - 1) + 1 for c, p in zip(self.subdomain_counts, self.nodes_per_subdomain))

    @property
    def spacing(self) -> tuple:
        return tuple(e / (n - 1) for e, n in zip(self.extents, self.global_shape))


@dataclass(frozen=True)
class SubdomainInfo:
    alpha: tuple
    lo: tuple
    shape: tuple
    neighbors: dict = field(default_factory=dict)

    def slices(self):
        return tuple(slice(l, l + s) for l, s in zip(self.lo, self.shape))


@dataclass(frozen=True)
class DomainPartition:
    spec: DomainSpec
    subdomains: tuple

    @property
    def global_shape(self):
        return self.spec.global_shape

    @property
    def spacing(self):
        return self.spec.spacing

    def subdomain(self, alpha) -> SubdomainInfo:
        cx, cy, cz = self.spec.subdomain_counts
        i, j, k = alpha
        if not (0 <= i < cx and 0 <= j < cy and 0 <= k < cz):
            raise KeyError(f"no subdomain {alpha}")
        return self.subdomains[(i * cy + j) * cz + k]


def build_partition(spec: DomainSpec) -> DomainPartition:
    """Tile the grid (grid.py:202-226); neighbours keyed by face id."""
    counts, p = spec.subdomain_counts, spec.nodes_per_subdomain
    subs = []
    for alpha in np.ndindex(*counts):
        alpha = tuple(int(a) for a in alpha)
        nb = {}
        for f in range(6):
            b = list(alpha)
            b[FACE_AXIS[f]] += 1 if FACE_SIDE[f] else -1
            if 0 <= b[FACE_AXIS[f]] < counts[FACE_AXIS[f]]:
                nb[f] = tuple(b)
        subs.append(SubdomainInfo(alpha, tuple(a * (q - 1) for a, q in zip(alpha, p)), tuple(p), nb))
    return DomainPartition(spec, tuple(subs))


@dataclass(frozen=True)
class FaceNodes:
    face: int
    indices: np.ndarray
    plane_shape: tuple
    lo: tuple = ()   # window start along the two in-plane axes
    hi: tuple = ()   # window end (exclusive)


def face_window(shape, face: int, neighbor_faces) -> FaceNodes:
    """Boundary window owned by ``face`` (ownership rule of grid.py:256-271, 385-412)."""
    ax = FACE_AXIS[face]
    layer = shape[ax] - 1 if FACE_SIDE[face] else 0
    mine = face in neighbor_faces
    axes, lo_hi = [], []
    for a in range(3):
        if a == ax:
            axes.append(np.array([layer]))
            continue
        lo, hi = 0, shape[a]
        if ((2 * a) in neighbor_faces) != mine:
            lo = 1 if (2 * a) in neighbor_faces else 0
        elif a < ax:
            lo = 1
        if ((2 * a + 1) in neighbor_faces) != mine:
            hi = shape[a] - 1 if (2 * a + 1) in neighbor_faces else shape[a]
        elif a < ax:
            hi = shape[a] - 1
        axes.append(np.arange(lo, hi))
        lo_hi.append((lo, hi))
    g = np.meshgrid(*axes, indexing="ij")
    flat = np.ravel_multi_index(tuple(x.ravel() for x in g), tuple(shape)).astype(np.int64)
    return FaceNodes(face, flat, tuple(h - l for l, h in lo_hi), tuple(l for l, _ in lo_hi),
                     tuple(h for _, h in lo_hi))


def axis_multiplicity(n: int, shared_low: bool, shared_high: bool) -> np.ndarray:
    m = np.ones(n)
    if shared_low:
        m[0] = 2.0
    if shared_high:
        m[-1] = 2.0
    return m


@dataclass(frozen=True)
class SubdomainOperator:
    """Per-subdomain operator description (grid.py:278-314).  ``matrix`` is only
    built on request (host CSR, for tests); the GPU path uses the stencil."""

    alpha: tuple
    lo: tuple
    shape: tuple
    spacing: tuple
    matrix: object
    c: np.ndarray
    mu: np.ndarray
    neighbors: dict
    face_nodes: dict

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.shape))

    def local_index(self, ijk_global) -> int:
        loc = tuple(g - l for g, l in zip(ijk_global, self.lo))
        if any(x < 0 or x >= s for x, s in zip(loc, self.shape)):
            raise KeyError(f"node {ijk_global} not in subdomain {self.alpha}")
        return int(np.ravel_multi_index(loc, self.shape))


def assemble_subdomain_operator(partition: DomainPartition, alpha, c_field: np.ndarray,
                                with_matrix: bool = False) -> SubdomainOperator:
    sub = partition.subdomain(alpha)
    shape = sub.shape
    c_loc = np.ascontiguousarray(c_field[sub.slices()], dtype=float)
    am = [axis_multiplicity(shape[a], (2 * a) in sub.neighbors, (2 * a + 1) in sub.neighbors)
          for a in range(3)]
    mult = (am[0][:, None, None] * am[1][None, :, None] * am[2][None, None, :]).ravel()
    faces = {f: face_window(shape, f, sub.neighbors) for f in range(6)}
    mat = None
    if with_matrix:
        mat = _stiffness_csr(shape, partition.spacing, c_loc, am)
    return SubdomainOperator(alpha, sub.lo, shape, partition.spacing, mat, c_loc.ravel(), 1.0 / mult,
                             dict(sub.neighbors), faces)


def _stiffness_csr(shape, spacing, c_loc, am):
    """Host CSR of A = D K D (grid.py:326-382, 438-445) -- tests/diagnostics only."""
    from scipy import sparse
    n = int(np.prod(shape))
    ids = np.arange(n).reshape(shape)
    rows, cols, vals = [], [], []
    diag = np.zeros(n)
    for d in range(3):
        a_sl = [slice(None)] * 3
        b_sl = [slice(None)] * 3
        a_sl[d] = slice(0, shape[d] - 1)
        b_sl[d] = slice(1, shape[d])
        i = ids[tuple(a_sl)].ravel()
        j = ids[tuple(b_sl)].ravel()
        ci = c_loc[tuple(a_sl)].ravel()
        cj = c_loc[tuple(b_sl)].ravel()
        wt = 1.0
        for a in range(3):
            if a != d:
                sh = [1, 1, 1]
                sh[a] = shape[a]
                wt = wt * am[a].reshape(sh)
        wt = np.broadcast_to(wt, [shape[a] - (a == d) for a in range(3)]).ravel()
        s = 1.0 / (wt * spacing[d] ** 2)
        rows += [i, j]
        cols += [j, i]
        vals += [ci * cj * s, ci * cj * s]
        np.add.at(diag, i, -ci * ci * s)
        np.add.at(diag, j, -cj * cj * s)
    rows.append(np.arange(n))
    cols.append(np.arange(n))
    vals.append(diag)
    k = sparse.coo_array((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    mult = (am[0][:, None, None] * am[1][None, :, None] * am[2][None, None, :]).ravel()
    dm = sparse.diags_array(np.sqrt(mult))
    mat = (dm @ k.tocsr() @ dm).tocsr()
    mat.sum_duplicates()
    return mat


def assemble_global_operator(partition: DomainPartition, c_field: np.ndarray):
    """Undivided operator ``C Lap_h C`` on the full grid, mirror closure (grid.py:461-467).

    Returns a matrix-free :class:`~paper_1406_6923_b200.fdtd.FineGridOperator`
    (``a @ x`` and the fine-grid solver run on the GPU) instead of a host CSR.
    """
    from .fdtd import FineGridOperator
    return FineGridOperator(partition.global_shape, partition.spacing, c_field)
