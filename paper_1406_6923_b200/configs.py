"""Seeded synthetic workloads for BASELINE.json configs 1-5.

The paper's own medium is unpublished (reference SPEC.md:604), so these
seeded fields stand in for it.  Conventions:

* every "16^3-node subdomain" is P = 17 nodes per edge sharing one node
  layer with each neighbour (reference grid.py:1-6, 76-85), h = 10 m, so the
  global grid has 16*C_a + 1 nodes per axis;
* shift s = (2 pi f0)^2 in SI units (the reference default 4.0 is
  dimensionless, sim.py:166);
* the Ricker source (sim.py:80-85, delay 1.2/f0 per sim.py:69) sits at node
  (G_a - 1)/2 - 1 per axis -- the exact centre is an interface node, which
  the reference rejects (sim.py:405-419);
* receivers: all layer-1 face coefficients of the z-midplane interfaces
  (face 5 of every subdomain with alpha_z = C_z/2 - 1), plus, for configs
  2-5, 8 node receivers along x through the source's (y, z).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED = 1406
P_NODES = 17
H = 10.0


@dataclass
class Workload:
    name: str
    counts: tuple
    p: tuple
    spacing: tuple
    c_field: np.ndarray
    modes_per_face: int
    n: int
    shift: float
    n_steps: int
    f0: float
    sources: list            # global node (i, j, k) per independent wavefield
    face_receivers: list     # (alpha, face) pairs; every mode of the face is recorded
    node_receivers: list     # global node (i, j, k)
    extra: dict = field(default_factory=dict)

    @property
    def global_shape(self):
        return tuple(c * (q - 1) + 1 for c, q in zip(self.counts, self.p))

    @property
    def n_sub(self):
        return int(np.prod(self.counts))

    @property
    def width(self):
        return 6 * self.modes_per_face

    @property
    def layers(self):
        return self.n + 1

    @property
    def delay(self):
        return 1.2 / self.f0


def _layered(rng, gshape, n_layers):
    ez = (gshape[2] - 1) * H
    v = rng.uniform(1500.0, 4500.0, size=n_layers)
    depths = np.sort(rng.uniform(0.25 * ez, 0.75 * ez, size=n_layers - 1))
    z = np.arange(gshape[2]) * H
    # inclusive boxes [d_k, E_z], later ones win (reference grid.py:88-100, 229-253)
    idx = np.zeros(gshape[2], dtype=int)
    for k, d in enumerate(depths):
        idx[z >= d] = k + 1
    col = v[idx]
    return np.broadcast_to(col[None, None, :], gshape).copy()


def _blocky(rng, gshape, cells):
    nb = [max(1, (g - 1) // cells) for g in gshape]
    vals = rng.uniform(1500.0, 4500.0, size=nb)
    ix = [np.minimum(np.arange(g) // cells, b - 1) for g, b in zip(gshape, nb)]
    return vals[np.ix_(*ix)]


def _midplane_receivers(counts):
    kz = counts[2] // 2 - 1
    if kz < 0:
        return []
    return [((i, j, kz), 5) for i in range(counts[0]) for j in range(counts[1])]


def _line_receivers(gshape, src):
    out = []
    for i in range(gshape[0]):
        if i % 16 == 8:
            out.append((i, src[1], src[2]))
    step = max(1, len(out) // 8)
    return out[::step][:8]


def source_node(gshape):
    return tuple((g - 1) // 2 - 1 for g in gshape)


def make_workload(cfg: int, counts=None, seed: int = SEED, n_steps=None) -> Workload:
    """Seeded workload for config ``cfg`` (1..5); ``counts`` shrinks the tiling
    for parity-sized runs while keeping the medium recipe and ROM parameters."""
    rng = np.random.default_rng(seed + cfg)
    base = {1: (2, 2, 2), 2: (8, 8, 8), 3: (16, 16, 16), 4: (16, 16, 16), 5: (32, 32, 16)}[cfg]
    counts = tuple(counts) if counts is not None else base
    p = (P_NODES,) * 3
    gshape = tuple(c * (P_NODES - 1) + 1 for c in counts)
    if cfg == 1:
        c = _layered(rng, gshape, 3)
        m, n, steps, f0 = 4, 4, 200, 15.0
    elif cfg == 2:
        c = _layered(rng, gshape, 5)
        g = np.array(gshape)
        while True:
            lo = np.array([rng.integers(1, max(2, gi - 26) + 1) for gi in g])
            hi = lo + 24
            if all(any(lo_a < 16 * q < hi_a for q in range(1, ca)) for lo_a, hi_a, ca
                   in zip(lo, hi, counts)) or min(counts) == 1:
                break
        hi = np.minimum(hi, g - 1)
        c[lo[0]:hi[0] + 1, lo[1]:hi[1] + 1, lo[2]:hi[2] + 1] = 5000.0
        m, n, steps, f0 = 4, 6, 1000, 15.0
    elif cfg in (3, 4):
        c = _blocky(rng, gshape, 8)
        m, n, steps, f0 = 9, 8, 2000, 10.0
    elif cfg == 5:
        c = _blocky(rng, gshape, 4)
        for _ in range(10):
            side = rng.integers(8, 41, size=3)
            lo = np.array([rng.integers(0, gi) for gi in gshape])
            hi = np.minimum(lo + side - 1, np.array(gshape) - 1)
            c[lo[0]:hi[0] + 1, lo[1]:hi[1] + 1, lo[2]:hi[2] + 1] = 5500.0
        m, n, steps, f0 = 9, 8, 4000, 10.0
    else:
        raise ValueError(f"unknown config {cfg}")
    src = source_node(gshape)
    sources = [src]
    if cfg == 4:
        srng = np.random.default_rng(seed + 400)
        sources = []
        while len(sources) < 32:
            ijk = tuple(int(srng.integers(0, g)) for g in gshape)
            if any(x % 16 == 0 for x in ijk):
                continue
            sources.append(ijk)
    node_rx = [] if cfg == 1 else _line_receivers(gshape, src)
    return Workload(
        name=f"config{cfg}" + ("" if counts == base else "-" + "x".join(map(str, counts))),
        counts=counts, p=p, spacing=(H, H, H), c_field=np.ascontiguousarray(c, dtype=float),
        modes_per_face=m, n=n, shift=(2.0 * math.pi * f0) ** 2,
        n_steps=steps if n_steps is None else n_steps, f0=f0,
        sources=sources, face_receivers=_midplane_receivers(counts), node_receivers=node_rx,
    )


def locate(ijk, counts, p):
    """(alpha, local row) of a strictly interior global node (sim.py:405-419)."""
    alpha, loc = [], []
    for x, c, q in zip(ijk, counts, p):
        a = min(x // (q - 1), c - 1)
        alpha.append(a)
        loc.append(x - a * (q - 1))
    return tuple(alpha), int(np.ravel_multi_index(tuple(loc), tuple(p)))
