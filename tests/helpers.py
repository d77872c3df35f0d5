"""Shared test helpers: golden fixtures -> product models, oracle runs."""

from __future__ import annotations

import os

import numpy as np

from paper_1406_6923_b200 import grid as pg
from paper_1406_6923_b200.rom import SubdomainModel

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    return np.load(os.path.join(GOLD, name))


def rel(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def partition_for(counts, p, extents):
    return pg.build_partition(pg.DomainSpec(tuple(extents), tuple(counts), tuple(p)))


def models_from_arrays(part, c_field, m, gammas, hats, scales, shift=0.0, basis=None, tdiag=None, toff=None):
    """SubdomainModel per alpha (sorted order) from stacked coefficient arrays."""
    out = {}
    order = sorted(s.alpha for s in part.subdomains)
    for i, a in enumerate(order):
        op = pg.assemble_subdomain_operator(part, a, c_field)
        out[a] = SubdomainModel(
            alpha=a, lo=op.lo, shape=op.shape, spacing=op.spacing, modes_per_face=m,
            layers=int(gammas[i].shape[0]), shift=shift, neighbors=dict(op.neighbors),
            face_indices=tuple(op.face_nodes[f].indices for f in range(6)),
            gammas=np.asarray(gammas[i]), gamma_hats=np.asarray(hats[i]), scales=np.asarray(scales[i]),
            basis=None if basis is None else np.asarray(basis[i]), c=op.c, mu=op.mu,
            tdiag=None if tdiag is None else tdiag[i], toff=None if toff is None else toff[i])
    return out


def oracle_models(wl, alphas=None):
    """Oracle-built models (oracle.sfw_oracle.Model) for a configs.Workload."""
    from oracle import sfw_oracle as so
    ops = so.make_subops(wl.counts, wl.p, wl.spacing, wl.c_field, alphas=alphas)
    return {a: so.build_model(ops[a], wl.modes_per_face, wl.n, wl.shift) for a in sorted(ops)}


def face_probes(models, wl):
    """Unit-weight probes on every mode of the configured receiver faces."""
    out = []
    for alpha, face in wl.face_receivers:
        md = models[alpha]
        for q in range(wl.modes_per_face):
            wts = np.zeros(md.state_size)
            wts[face * wl.modes_per_face + q] = 1.0
            out.append((alpha, wts))
    return out


def batched_oracle(models, dt, sources=(), m=None, alt=False):
    """oracle.CoupledBatched over product models (uniform layers), plus the alpha -> index map.
    ``sources``: SourceTerm-like objects (alpha, vector, profile).  ``alt``: einsum products in
    place of BLAS, i.e. another summation order -- the oracle's own rounding floor."""
    from oracle import sfw_oracle as so
    order = sorted(models)
    idx = {a: i for i, a in enumerate(order)}
    nbr = np.full((len(order), 6), -1, dtype=np.int64)
    for a in order:
        for f, b in models[a].neighbors.items():
            nbr[idx[a], f] = idx[b]
    G = np.stack([np.asarray(models[a].gammas) for a in order])
    H = np.stack([np.asarray(models[a].gamma_hats) for a in order])
    m = m or models[order[0]].modes_per_face
    src = [(idx[s.alpha], s.vector, s.profile) for s in sources]
    return so.CoupledBatched(G, H, nbr, m, dt, sources=src, alt=alt), idx

