"""CPU oracle for the S-fraction ROM path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference `sfwave` package's
two hot-path stages (reference = /root/reference/pkg/src/sfwave, read-only,
not present on GPU boxes).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it,
and only as the checker or the timed CPU baseline.  The product path
(``paper_1406_6923_b200``) never imports it.

Parity pin: every function below is checked against golden vectors produced
by the reference itself (``tests/golden/make_golden.py`` imports the real
``sfwave`` in the build container and commits ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` compares).

Algorithm map (reference file:line it restates):

* geometry / operator ........ grid.py:76-85, 202-226, 317-458
* face inputs ................ rom.py:45-86
* shifted-inverse Krylov ..... rom.py:89-174  (scipy SuperLU, CGS2, pivoted QR)
* truncation + projection .... rom.py:177-182, 359-434
* block Lanczos .............. rom.py:202-262
* S-fraction recursion ....... rom.py:265-316
* source / probe maps ........ stepper.py:91-141
* coupled leapfrog ........... stepper.py:178-415
* energy ..................... stepper.py:419-449
* coupled CFL power iteration  stepper.py:452-495, reference.py:20-23
* Ricker pulse ............... sim.py:80-85
* fine-grid operator / FDTD .. grid.py:461-467, reference.py:26-157
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
from scipy.sparse.linalg import splu

# reference.py:20-23 / rom.py:38-42
POWER_TOL = 1e-8
POWER_MAX_ITER = 10000
CFL_SAFETY = 0.9
GROWTH_LIMIT = 1e6
DEFLATION_RTOL = 1e-12
CONDITION_LIMIT = 1e12


class OracleError(Exception):
    """Raised where the reference raises NumericalError/ConfigError/...

    ``kind`` names the reference exception class so tests can compare the
    error taxonomy (errors.py:11-41).
    """

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# ---------------------------------------------------------------------------
# geometry (grid.py:76-85, 202-226, 317-412)

def global_shape(counts, p):
    return tuple(c * (n - 1) + 1 for c, n in zip(counts, p))


def neighbor_faces(alpha, counts):
    """Face ids 0..5 (-x,+x,-y,+y,-z,+z) that have a neighbour (grid.py:212-217)."""
    out = {}
    for f in range(6):
        ax, hi = f // 2, f % 2
        b = list(alpha)
        b[ax] += 1 if hi else -1
        if 0 <= b[ax] < counts[ax]:
            out[f] = tuple(b)
    return out


def _mult_1d(n, lo_shared, hi_shared):
    m = np.ones(n)
    if lo_shared:
        m[0] = 2.0
    if hi_shared:
        m[-1] = 2.0
    return m


def face_window(shape, face, nbr):
    """(flat indices, plane_shape) of the boundary window owned by ``face``.

    Ownership rule of grid.py:385-412: an edge lying on two face planes goes
    to the interface plane when exactly one of them is an interface,
    otherwise to the plane with the smaller normal axis.
    """
    ax = face // 2
    layer = shape[ax] - 1 if face % 2 else 0
    own_is_iface = face in nbr
    axes = []
    for a in range(3):
        if a == ax:
            axes.append(np.array([layer]))
            continue
        lo, hi = 0, shape[a]
        for side in (0, 1):
            other_is_iface = (2 * a + side) in nbr
            drop = other_is_iface if other_is_iface != own_is_iface else (a < ax)
            if drop:
                if side:
                    hi -= 1
                else:
                    lo += 1
        axes.append(np.arange(lo, hi))
    g = np.meshgrid(*axes, indexing="ij")
    flat = np.ravel_multi_index(tuple(x.ravel() for x in g), shape).astype(np.int64)
    dims = tuple(len(axes[a]) for a in range(3) if a != ax)
    return flat, dims


def subdomain_matrix(shape, spacing, c_loc, nbr):
    """Weighted operator A = D K D of one subdomain (grid.py:326-382, 415-458).

    K sums, over every grid link e=(i,j), -(c_i e_i - c_j e_j)(...)^T / (w_e h^2)
    where w_e is the product of the transverse sharing multiplicities;
    D = diag(sqrt(mult)).  Returns (csr matrix, mu = 1/mult).
    """
    n = int(np.prod(shape))
    cv = np.asarray(c_loc, float).reshape(shape)
    mults = [_mult_1d(shape[a], (2 * a) in nbr, (2 * a + 1) in nbr) for a in range(3)]
    ids = np.arange(n).reshape(shape)
    r_all, c_all, v_all = [], [], []
    diag = np.zeros(n)
    for d in range(3):
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[d] = slice(0, shape[d] - 1)
        hi[d] = slice(1, shape[d])
        i = ids[tuple(lo)].ravel()
        j = ids[tuple(hi)].ravel()
        ci = cv[tuple(lo)].ravel()
        cj = cv[tuple(hi)].ravel()
        wt = np.ones([shape[a] if a != d else shape[d] - 1 for a in range(3)])
        for a in range(3):
            if a != d:
                bshape = [1, 1, 1]
                bshape[a] = shape[a]
                wt = wt * mults[a].reshape(bshape)
        s = 1.0 / (wt.ravel() * spacing[d] ** 2)
        off = ci * cj * s
        r_all += [i, j]
        c_all += [j, i]
        v_all += [off, off]
        np.add.at(diag, i, -ci * ci * s)
        np.add.at(diag, j, -cj * cj * s)
    r_all.append(np.arange(n))
    c_all.append(np.arange(n))
    v_all.append(diag)
    k = sp.coo_array((np.concatenate(v_all), (np.concatenate(r_all), np.concatenate(c_all))),
                     shape=(n, n)).tocsr()
    mult = (mults[0][:, None, None] * mults[1][None, :, None] * mults[2][None, None, :]).ravel()
    dmat = sp.diags_array(np.sqrt(mult))
    a = (dmat @ k @ dmat).tocsr()
    a.sum_duplicates()
    return a, 1.0 / mult


@dataclass
class SubOp:
    """Per-subdomain operator bundle (mirrors grid.py:278-306 SubdomainOperator)."""

    alpha: tuple
    lo: tuple
    shape: tuple
    spacing: tuple
    matrix: object
    c: np.ndarray
    mu: np.ndarray
    neighbors: dict
    faces: list  # [(indices, plane_shape)] * 6


def make_subops(counts, p, spacing, c_field, alphas=None):
    """Operators for every (or the listed) subdomain of a tiling."""
    out = {}
    every = [(i, j, k) for i in range(counts[0]) for j in range(counts[1]) for k in range(counts[2])]
    for alpha in (every if alphas is None else alphas):
        lo = tuple(a * (n - 1) for a, n in zip(alpha, p))
        sl = tuple(slice(l, l + n) for l, n in zip(lo, p))
        c_loc = np.ascontiguousarray(c_field[sl], dtype=float)
        nbr = neighbor_faces(alpha, counts)
        mat, mu = subdomain_matrix(tuple(p), tuple(spacing), c_loc, nbr)
        faces = [face_window(tuple(p), f, nbr) for f in range(6)]
        out[alpha] = SubOp(alpha, lo, tuple(p), tuple(spacing), mat, c_loc.ravel(), mu, nbr, faces)
    return out


# ---------------------------------------------------------------------------
# offline ROM build (rom.py:45-434)

def dct2_modes(n, k):
    """First k orthonormal DCT-II vectors on n samples (rom.py:45-52)."""
    x = (np.arange(n, dtype=float) + 0.5)[:, None] * np.arange(k, dtype=float)[None, :]
    out = np.cos(np.pi * x / n)
    sc = np.full(k, math.sqrt(2.0 / n))
    sc[0] = math.sqrt(1.0 / n)
    return out * sc


def face_inputs(op: SubOp, m):
    """Input block F (N x 6m), face f in columns [f m, (f+1) m) (rom.py:55-86)."""
    k = math.isqrt(m)
    if k * k != m:
        raise OracleError("ConfigError", f"modes per face must be a perfect square, got {m}")
    n = int(np.prod(op.shape))
    f = np.zeros((n, 6 * m))
    for fid, (idx, (na, nb)) in enumerate(op.faces):
        if k > na or k > nb:
            raise OracleError("ConfigError", "face window too small for the mode count")
        f[idx, fid * m:(fid + 1) * m] = np.kron(dct2_modes(na, k), dct2_modes(nb, k))
    return f


def _solver(matrix, shift):
    """x -> (A - sI)^-1 x via one SuperLU factor of -A + sI (rom.py:89-116)."""
    n = matrix.shape[0]
    work = (-matrix + shift * sp.identity(n, format="csc")).tocsc()
    try:
        lu = splu(work)
    except RuntimeError as exc:
        raise OracleError("NumericalError", f"factorization of the shifted operator failed ({exc})")
    return lambda x: -lu.solve(x)


def _orth_against(basis, raw, rtol):
    """CGS2 against basis, then pivoted-QR deflation with sign gauge (rom.py:119-136)."""
    x = raw.copy()
    x -= basis @ (basis.T @ x)
    x -= basis @ (basis.T @ x)
    tol = rtol * max(float(np.linalg.norm(raw)), 1e-300)
    q, r, _ = sla.qr(x, mode="economic", pivoting=True)
    d = np.diag(r)
    rank = int(np.sum(np.abs(d) > tol))
    if rank == 0:
        return x[:, :0]
    sg = np.sign(d[:rank])
    sg[sg == 0] = 1.0
    return q[:, :rank] * sg


def krylov_basis(matrix, f, n, shift, rtol=DEFLATION_RTOL):
    """V spanning {F, (A-sI)^-1 F, ..., (A-sI)^-n F}; returns (V, block sizes) (rom.py:139-174)."""
    if np.linalg.norm(f.T @ f - np.eye(f.shape[1])) > 1e-10:
        raise OracleError("NumericalError", "input block must be orthonormal")
    solve = _solver(matrix, shift)
    cols = [f]
    sizes = [f.shape[1]]
    v = f.copy()
    prev = f
    for _ in range(n):
        nxt = _orth_against(v, solve(prev), rtol)
        if nxt.shape[1] == 0:
            sizes.append(0)
            break
        v = np.hstack([v, nxt])
        sizes.append(nxt.shape[1])
        prev = nxt
    return v, sizes


def galerkin(v, matrix, f):
    """(sym(V^T A V), V^T F) (rom.py:177-182)."""
    at = v.T @ (matrix @ v)
    return 0.5 * (at + at.T), v.T @ f


def _qr_pos(z):
    q, r = np.linalg.qr(z)
    sg = np.sign(np.diag(r))
    sg[sg == 0] = 1.0
    return q * sg, r * sg[:, None]


@dataclass
class Chain:
    diag: list
    off: list
    entry: np.ndarray
    q: np.ndarray
    sizes: list = field(default_factory=list)


def lanczos(at, ft):
    """Block Lanczos with full two-pass reorthogonalisation (rom.py:202-262)."""
    dim, width = ft.shape
    tol = 1e-11 * max(float(np.linalg.norm(at)) / math.sqrt(dim), 1e-300)
    q1, b1 = _qr_pos(ft)
    qs = [q1]
    basis = q1
    diag, off = [], []
    sizes = [width]
    while True:
        qj = qs[-1]
        z = at @ qj
        if len(qs) > 1:
            z -= qs[-2] @ off[-1].T
        aj = qj.T @ z
        aj = 0.5 * (aj + aj.T)
        diag.append(aj)
        z -= qj @ aj
        z -= basis @ (basis.T @ z)
        z -= basis @ (basis.T @ z)
        if basis.shape[1] + z.shape[1] > dim and dim - basis.shape[1] <= 0:
            break
        qn, rn = np.linalg.qr(z)
        rank = int(np.sum(np.abs(np.diag(rn)) > tol))
        if rank < z.shape[1]:
            if rank > 0:
                sizes.append(rank)
            break
        sg = np.sign(np.diag(rn))
        sg[sg == 0] = 1.0
        off.append(rn * sg[:, None])
        qs.append(qn * sg)
        basis = np.hstack([basis, qs[-1]])
        sizes.append(z.shape[1])
    nl = len(diag)
    return Chain(diag, off[:nl - 1], b1, np.hstack(qs[:nl]), sizes[:nl])


def _congruence_inv(g, a):
    """sym(G^-T A G^-1) via two general solves (rom.py:265-269)."""
    y = np.linalg.solve(g.T, a)
    z = np.linalg.solve(g.T, y.T).T
    return 0.5 * (z + z.T)


def sfraction(diag, off, entry):
    """Chain coefficients (Gamma_j, Gamma-hat_j, G_j) (rom.py:272-316)."""
    nl = len(diag)
    w = entry.shape[0]
    gam, hat, scl = [], [], []
    g = entry.T.copy()
    gprev = np.zeros((w, w))
    for j in range(nl):
        if np.linalg.cond(g) > CONDITION_LIMIT:
            raise OracleError("NumericalError", f"chain scale matrix at layer {j + 1} is singular")
        scl.append(g)
        hat.append(g @ g.T)
        gj = -_congruence_inv(g, diag[j]) - gprev
        gam.append(gj)
        if j + 1 < nl:
            if np.linalg.cond(gj) > CONDITION_LIMIT:
                raise OracleError("NumericalError", f"chain link matrix at layer {j + 1} is singular")
            g = np.linalg.solve(g.T @ gj, off[j].T)
        gprev = gj
    return gam, hat, scl


@dataclass
class Model:
    """Mirror of rom.py:319-356 SubdomainModel (fields the path uses)."""

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

    @property
    def width(self):
        return 6 * self.modes_per_face

    def face_slice(self, f):
        m = self.modes_per_face
        return slice(f * m, (f + 1) * m)

    @property
    def state_size(self):
        return self.layers * self.width


def build_model(op: SubOp, m, n, shift):
    """Full offline pipeline for one subdomain (rom.py:359-434)."""
    w = 6 * m
    f = face_inputs(op, m)
    v, sizes = krylov_basis(op.matrix, f, n, shift)
    keep = 0
    for s in sizes:
        if s != w:
            break
        keep += 1
    if keep < 2:
        raise OracleError("NumericalError", f"subdomain {op.alpha}: dependent at depth 1 ({sizes})")
    truncated = keep < n + 1
    if truncated:
        v = v[:, :keep * w]
    at, ft = galerkin(v, op.matrix, f)
    ch = lanczos(at, ft)
    if ch.sizes != [w] * keep:
        raise OracleError("NumericalError", f"subdomain {op.alpha}: tridiagonalization lost rank")
    gam, hat, scl = sfraction(ch.diag, ch.off, ch.entry)
    if np.linalg.norm(hat[0] - np.eye(w)) > 1e-8:
        raise OracleError("NumericalError", "first inverse-mass block deviates from identity")
    return Model(
        alpha=op.alpha, lo=op.lo, shape=op.shape, spacing=op.spacing, modes_per_face=m,
        layers=keep, shift=shift, neighbors=dict(op.neighbors),
        face_indices=tuple(op.faces[f][0] for f in range(6)),
        gammas=np.stack(gam), gamma_hats=np.stack(hat), scales=np.stack(scl),
        basis=v @ ch.q, c=op.c, mu=op.mu, deflated=keep < len(sizes), truncated=truncated,
        tdiag=np.stack(ch.diag), toff=np.stack(ch.off) if ch.off else np.zeros((0, w, w)),
    )


# ---------------------------------------------------------------------------
# online maps (stepper.py:91-141)

def source_vector(model: Model, row, amplitude=1.0):
    """State-space forcing of a point source at a strictly interior node (stepper.py:91-128)."""
    if model.basis is None:
        raise OracleError("NumericalError", "model has no basis")
    if model.mu[row] < 1.0:
        raise OracleError("ConfigError", "source node lies on a subdomain interface")
    e = np.zeros(model.basis.shape[0])
    e[row] = amplitude / model.c[row]
    coeff = model.basis.T @ e
    w = model.width
    lead = float(np.linalg.norm(coeff[:w]))
    if lead > 1e-8 * max(float(np.linalg.norm(coeff)), 1e-300):
        raise OracleError("NumericalError", "interior source leaked into the boundary layer block")
    coeff[:w] = 0.0
    out = np.empty_like(coeff)
    for j in range(model.layers):
        s = slice(j * w, (j + 1) * w)
        out[s] = model.scales[j] @ coeff[s]
    return out


def probe_weights(model: Model, row):
    """Receiver functional for the physical field at a node (stepper.py:131-141)."""
    if model.basis is None:
        raise OracleError("NumericalError", "model has no basis")
    w = model.width
    out = np.empty(model.state_size)
    for j in range(model.layers):
        s = slice(j * w, (j + 1) * w)
        out[s] = np.linalg.solve(model.scales[j].T, model.basis[row, s])
    return out * (model.c[row] / np.sqrt(model.mu[row]))


def ricker(f_peak, delay):
    """sim.py:80-85."""
    def pulse(t):
        a = (math.pi * f_peak * (t - delay)) ** 2
        return (1.0 - 2.0 * a) * math.exp(-a)
    return pulse


# ---------------------------------------------------------------------------
# coupled leapfrog (stepper.py:178-449)

class Coupled:
    """Restatement of CoupledStepper with the same per-subdomain loop shape.

    sources: list of (alpha, vector, profile); probes: list of (alpha, weights).
    """

    def __init__(self, models: dict, dt: float, sources=()):
        if dt <= 0:
            raise OracleError("ConfigError", "time step must be positive")
        self.models = dict(models)
        self.order = sorted(self.models)
        self.dt = float(dt)
        self.sources = tuple(sources)
        for a, _, _ in self.sources:
            if a not in self.models:
                raise OracleError("ConfigError", f"source subdomain {a} has no model")
        self.ifaces = self._pair()
        self.message_count = 0
        self.steps_done = 0
        self.time = 0.0
        self.u_prev, self.u_curr = {}, {}
        self._base = 0.0

    def _pair(self):
        out = []
        for a in self.order:
            md = self.models[a]
            if np.linalg.norm(md.gamma_hats[0] - np.eye(md.width)) > 1e-8:
                raise OracleError("NumericalError", "first inverse-mass block is not the identity")
            for f, b in sorted(md.neighbors.items()):
                if b not in self.models:
                    raise OracleError("ProtocolError", f"missing neighbour {b}")
                other = self.models[b]
                if other.neighbors.get(f ^ 1) != a:
                    raise OracleError("ProtocolError", "inconsistent neighbour tables")
                if other.modes_per_face != md.modes_per_face:
                    raise OracleError("ProtocolError", "mode count mismatch")
                if a < b:
                    ha = md.gamma_hats[0][md.face_slice(f), md.face_slice(f)]
                    hb = other.gamma_hats[0][other.face_slice(f ^ 1), other.face_slice(f ^ 1)]
                    mass = ha @ np.linalg.solve(ha + hb, hb)
                    out.append((a, f, b, f ^ 1, 0.5 * (mass + mass.T)))
        return out

    def _flux(self, st, a):
        md = self.models[a]
        w = md.width
        u = st[a]
        u2 = u[w:2 * w] if md.layers > 1 else np.zeros(w)
        return md.gammas[0] @ (u2 - u[:w])

    def acceleration(self, st, count=False):
        flux = {a: self._flux(st, a) for a in self.order}
        inbox = {}
        for a in self.order:
            md = self.models[a]
            for f, b in sorted(md.neighbors.items()):
                inbox[(b, f ^ 1)] = flux[a][md.face_slice(f)]
                if count:
                    self.message_count += 1
        shared = {}
        for lo, lf, hi, hf, mass in self.ifaces:
            own = flux[lo][self.models[lo].face_slice(lf)]
            msg = inbox.get((lo, lf))
            if msg is None:
                raise OracleError("ProtocolError", "lost face message")
            seg = mass @ (own + msg)
            shared[(lo, lf)] = seg
            shared[(hi, hf)] = seg
        acc = {}
        for a in self.order:
            md = self.models[a]
            w, nl = md.width, md.layers
            u = st[a]
            out = np.empty_like(u)
            out[:w] = md.gamma_hats[0] @ flux[a]
            for f in md.neighbors:
                out[md.face_slice(f)] = shared[(a, f)]
            for j in range(1, nl):
                cur = u[j * w:(j + 1) * w]
                prv = u[(j - 1) * w:j * w]
                nxt = u[(j + 1) * w:(j + 2) * w] if j + 1 < nl else 0.0
                out[j * w:(j + 1) * w] = md.gamma_hats[j] @ (
                    md.gammas[j] @ (nxt - cur) - md.gammas[j - 1] @ (cur - prv))
            acc[a] = out
        return acc

    def _force(self, t):
        out = {}
        for a, vec, prof in self.sources:
            term = vec * prof(t)
            out[a] = out[a] + term if a in out else term
        return out

    def initialize(self, u0=None, v0=None):
        self.u_curr = {a: (np.array(u0[a], dtype=float) if u0 and a in u0
                           else np.zeros(self.models[a].state_size)) for a in self.order}
        vel = {a: (np.asarray(v0[a], dtype=float) if v0 and a in v0
                   else np.zeros(self.models[a].state_size)) for a in self.order}
        acc = self.acceleration(self.u_curr)
        frc = self._force(0.0)
        dt = self.dt
        self.u_prev = {a: self.u_curr[a] - dt * vel[a] + 0.5 * dt * dt * (acc[a] + frc.get(a, 0.0))
                       for a in self.order}
        self.steps_done = 0
        self.time = 0.0
        self.message_count = 0
        self._base = sum(float(np.linalg.norm(self.u_curr[a])) + dt * float(np.linalg.norm(vel[a]))
                         for a in self.order)

    def advance(self):
        dt = self.dt
        t = self.time
        acc = self.acceleration(self.u_curr, count=True)
        frc = self._force(t)
        nxt = {a: 2.0 * self.u_curr[a] - self.u_prev[a] + dt * dt * (acc[a] + frc.get(a, 0.0))
               for a in self.order}
        self.u_prev, self.u_curr = self.u_curr, nxt
        self.steps_done += 1
        self.time = self.steps_done * dt
        for _, vec, prof in self.sources:
            self._base += dt * dt * abs(float(prof(t))) * float(np.linalg.norm(vec))
        nrm = np.sqrt(sum(float(u @ u) for u in self.u_curr.values()))
        if nrm > GROWTH_LIMIT * max(self._base, 1e-300):
            raise OracleError("InstabilityError", f"coupled stepping diverged at step {self.steps_done}")

    def run(self, n_steps, probes=(), record_every=1, u0=None, v0=None):
        self.initialize(u0, v0)
        times = [0.0]
        rows = [self._row(probes)]
        for step in range(1, n_steps + 1):
            self.advance()
            if step % record_every == 0:
                times.append(self.time)
                rows.append(self._row(probes))
        return np.asarray(times), np.asarray(rows)

    def _row(self, probes):
        return np.array([wts @ self.u_curr[a] for a, wts in probes])

    def energy(self):
        dt = self.dt
        tot = 0.0
        for a in self.order:
            md = self.models[a]
            w, nl = md.width, md.layers
            diff = (self.u_curr[a] - self.u_prev[a]) / dt
            for j in range(nl):
                y = np.linalg.solve(md.scales[j], diff[j * w:(j + 1) * w])
                tot += 0.5 * float(y @ y)
            for j in range(nl):
                s = slice(j * w, (j + 1) * w)
                if j + 1 < nl:
                    s2 = slice((j + 1) * w, (j + 2) * w)
                    da = self.u_curr[a][s2] - self.u_curr[a][s]
                    db = self.u_prev[a][s2] - self.u_prev[a][s]
                else:
                    da = -self.u_curr[a][s]
                    db = -self.u_prev[a][s]
                tot += 0.5 * float(da @ (md.gammas[j] @ db))
        return tot


class CoupledBatched:
    """``Coupled`` restated over stacked arrays, for full-size (4096 / 16384-subdomain) windows.

    Same formulas and evaluation order per subdomain as ``Coupled`` (stepper.py:243-389):
    flux_1 = Gamma_1 (U_2 - U_1); acc_1 = Gamma-hat_1 flux_1 with shared face slices replaced by
    mass (own + msg); acc_j = Gamma-hat_j (Gamma_j (U_{j+1} - U_j) - Gamma_{j-1} (U_j - U_{j-1}));
    U_next = 2 U - U_prev + dt^2 (acc + f).  The block products are numpy stacked matmuls instead
    of per-subdomain gemv calls, so it agrees with ``Coupled`` to rounding (tests/test_oracle_golden.py
    pins the two against each other), not bit for bit.  Uniform layer count only.

    gammas / hats: (n, L, w, w) in sorted(alpha) order; nbr: (n, 6) neighbour index or -1;
    sources: list of (index, vector, profile); probes: list of (index, weights).
    """

    def __init__(self, gammas, hats, nbr, m, dt, sources=(), alt=False):
        self.alt = bool(alt)  # einsum products: another summation order (measures the oracle's floor)
        self.G = np.asarray(gammas, dtype=float)
        self.H = np.asarray(hats, dtype=float)
        self.n, self.L, self.w = self.G.shape[0], self.G.shape[1], self.G.shape[2]
        self.m = int(m)
        self.nbr = np.asarray(nbr, dtype=np.int64)
        self.dt = float(dt)
        self.sources = tuple(sources)
        lo, lf, hi, hf, mass = [], [], [], [], []
        for a in range(self.n):  # stepper.py:178-220 pairing, low index owns the interface
            for f in range(6):
                b = int(self.nbr[a, f])
                if b > a:
                    sa = slice(f * m, (f + 1) * m)
                    sb = slice((f ^ 1) * m, ((f ^ 1) + 1) * m)
                    ha = self.H[a, 0][sa, sa]
                    hb = self.H[b, 0][sb, sb]
                    mm = ha @ np.linalg.solve(ha + hb, hb)
                    lo.append(a)
                    lf.append(f)
                    hi.append(b)
                    hf.append(f ^ 1)
                    mass.append(0.5 * (mm + mm.T))
        self.if_lo, self.if_lf = np.array(lo, dtype=np.int64), np.array(lf, dtype=np.int64)
        self.if_hi, self.if_hf = np.array(hi, dtype=np.int64), np.array(hf, dtype=np.int64)
        self.mass = np.stack(mass) if mass else np.zeros((0, m, m))
        self._fidx = np.arange(m)
        self.steps_done = 0
        self.time = 0.0
        self._base = 0.0

    def _mv(self, A, x):
        if self.alt:
            return np.einsum("nij,nj->ni", A, x)
        return np.matmul(A, x[..., None])[..., 0]

    def acceleration(self, U):
        """U: (n, L, w) -> acc (n, L, w)."""
        m, L = self.m, self.L
        u2 = U[:, 1] if L > 1 else np.zeros_like(U[:, 0])
        flux = self._mv(self.G[:, 0], u2 - U[:, 0])
        acc = np.empty_like(U)
        acc[:, 0] = self._mv(self.H[:, 0], flux)
        if len(self.if_lo):
            cols_lo = self.if_lf[:, None] * m + self._fidx[None, :]
            cols_hi = self.if_hf[:, None] * m + self._fidx[None, :]
            own = flux[self.if_lo[:, None], cols_lo]
            msg = flux[self.if_hi[:, None], cols_hi]
            seg = self._mv(self.mass, own + msg)
            acc[self.if_lo[:, None], 0, cols_lo] = seg
            acc[self.if_hi[:, None], 0, cols_hi] = seg
        for j in range(1, L):
            cur, prv = U[:, j], U[:, j - 1]
            nxt = U[:, j + 1] if j + 1 < L else 0.0
            acc[:, j] = self._mv(self.H[:, j], self._mv(self.G[:, j], nxt - cur) - self._mv(self.G[:, j - 1], cur - prv))
        return acc

    def _force(self, t):
        out = {}
        for i, vec, prof in self.sources:
            term = np.asarray(vec, dtype=float).reshape(self.L, self.w) * prof(t)
            out[i] = out[i] + term if i in out else term
        return out

    def initialize(self, u0=None, v0=None):
        self.u_curr = np.zeros((self.n, self.L, self.w)) if u0 is None else np.array(u0, dtype=float)
        vel = np.zeros_like(self.u_curr) if v0 is None else np.asarray(v0, dtype=float)
        acc = self.acceleration(self.u_curr)
        for i, f in self._force(0.0).items():
            acc[i] = acc[i] + f
        dt = self.dt
        self.u_prev = self.u_curr - dt * vel + 0.5 * dt * dt * acc
        self.steps_done = 0
        self.time = 0.0
        self._base = float(np.sum(np.linalg.norm(self.u_curr.reshape(self.n, -1), axis=1))
                           + dt * np.sum(np.linalg.norm(vel.reshape(self.n, -1), axis=1)))

    def advance(self):
        dt = self.dt
        t = self.time
        acc = self.acceleration(self.u_curr)
        for i, f in self._force(t).items():
            acc[i] = acc[i] + f
        nxt = 2.0 * self.u_curr - self.u_prev + dt * dt * acc
        self.u_prev, self.u_curr = self.u_curr, nxt
        self.steps_done += 1
        self.time = self.steps_done * dt
        for _, vec, prof in self.sources:
            self._base += dt * dt * abs(float(prof(t))) * float(np.linalg.norm(vec))
        nrm = float(np.sqrt(np.sum(self.u_curr * self.u_curr)))
        if nrm > GROWTH_LIMIT * max(self._base, 1e-300):
            raise OracleError("InstabilityError", f"coupled stepping diverged at step {self.steps_done}")

    def run(self, n_steps, probes=(), u0=None, v0=None):
        self.initialize(u0, v0)
        pi = np.array([i for i, _ in probes], dtype=np.int64)
        pw = np.stack([np.asarray(wt, dtype=float) for _, wt in probes]) if probes else np.zeros((0, self.L * self.w))

        def row():
            return np.einsum("pk,pk->p", pw, self.u_curr.reshape(self.n, -1)[pi]) if len(pi) else np.zeros(0)

        rows = [row()]
        for _ in range(n_steps):
            self.advance()
            rows.append(row())
        return np.arange(n_steps + 1) * self.dt, np.asarray(rows)


def cfl_power(models: dict, tol=POWER_TOL, max_iter=POWER_MAX_ITER, seed=0):
    """(lambda_hat, converged) of the coupled map (stepper.py:452-487)."""
    st = Coupled(models, dt=1.0)
    rng = np.random.default_rng(seed)
    x = {a: rng.standard_normal(models[a].state_size) for a in st.order}

    def unit(vec):
        nrm = np.sqrt(sum(float(v @ v) for v in vec.values()))
        return {a: v / nrm for a, v in vec.items()}, nrm

    x, _ = unit(x)
    lam = 0.0
    for it in range(max_iter):
        neg = st.acceleration(x)
        y = {a: -neg[a] for a in neg}
        lam_new = sum(float(x[a] @ y[a]) for a in y)
        y, nrm = unit(y)
        if nrm == 0.0:
            return 0.0, True
        if it > 0 and abs(lam_new - lam) <= tol * abs(lam_new):
            return lam_new, True
        lam = lam_new
        x = y
    return lam, False


# ---------------------------------------------------------------------------
# fine-grid reference solver (grid.py:461-467, reference.py:26-157)

def global_matrix(shape, spacing, c_field):
    """Undivided C Lap_h C on the full grid (grid.py:461-467): subdomain_matrix with no sharing."""
    a, _ = subdomain_matrix(tuple(shape), tuple(spacing), np.asarray(c_field, float).ravel(), {})
    return a


def power_lambda(a, tol=POWER_TOL, max_iter=POWER_MAX_ITER, seed=0):
    """(lambda_max(-A), iterations) by power iteration (reference.py:26-63)."""
    n = a.shape[0]
    v = np.random.default_rng(seed).standard_normal(n)
    v /= np.linalg.norm(v)
    lam = 0.0
    for it in range(max_iter):
        w = -(a @ v)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0, it + 1
        lam_new = float(v @ w)
        v = w / nw
        if it > 0 and abs(lam_new - lam) <= tol * abs(lam_new):
            return lam_new, it + 1
        lam = lam_new
    return lam, -max_iter


def leapfrog(a, dt, n_steps, u0=None, v0=None, source_vec=None, source_fn=None, record_idx=None,
             record_every=1, damping=None, growth_limit=GROWTH_LIMIT):
    """Central-difference integration of w_tt = A w + f(t) s (reference.py:86-157).

    Returns (samples, times, u_prev, u_curr); raises OracleError on growth.
    """
    n = a.shape[0]
    u = np.zeros(n) if u0 is None else np.array(u0, dtype=float)
    vel = np.zeros(n) if v0 is None else np.asarray(v0, dtype=float)
    forced = source_vec is not None and source_fn is not None
    snorm = float(np.linalg.norm(source_vec)) if forced else 0.0

    def acc_of(x, t):
        y = a @ x
        return y + source_fn(t) * source_vec if forced else y

    up = u - dt * vel + 0.5 * dt * dt * acc_of(u, 0.0)
    rec = None if record_idx is None else np.asarray(record_idx, dtype=np.int64)
    samples, times = ([u[rec].copy()], [0.0]) if rec is not None else ([], [])
    base = float(np.linalg.norm(u)) + dt * float(np.linalg.norm(vel))
    for step in range(1, n_steps + 1):
        t = (step - 1) * dt
        un = 2.0 * u - up + dt * dt * acc_of(u, t)
        if damping is not None:
            un = un * damping
        up, u = u, un
        if forced:
            base += dt * dt * abs(float(source_fn(t))) * snorm
        if float(np.linalg.norm(u)) > growth_limit * max(base, 1e-300):
            raise OracleError(f"leapfrog diverged at step {step}")
        if rec is not None and step % record_every == 0:
            samples.append(u[rec].copy())
            times.append(step * dt)
    return np.array(samples), np.array(times), up, u
