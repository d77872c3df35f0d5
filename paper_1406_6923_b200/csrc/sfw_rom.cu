// Stage 1: batched off-line ROM build on sm_100a.
//
// Replaces reference rom.py:359-434 (build_subdomain_model) and its pieces,
// run for a whole batch of subdomains at once:
//   face inputs F            rom.py:45-86      k_face_basis
//   (A - sI)^-1 solves       rom.py:89-116     k_pcg  (see below)
//   CGS2 + QR deflation      rom.py:119-136    DMMA GEMMs + k_cholqr (CholQR2)
//   Krylov loop              rom.py:139-174
//   Galerkin projection      rom.py:177-182    k_stencil + DMMA GEMM
//   block Lanczos            rom.py:202-262    DMMA GEMMs + k_cholqr
//   S-fraction recursion     rom.py:265-316    k_sfraction (smem LU / Jacobi SVD)
//
// The shifted solve.  The subdomain operator of reference grid.py:415-458 is
// A = D K D with K the link-weighted C Lap C; it factors exactly as
//     A = -C S C,   S = X_x (+) X_y (+) X_z   (Kronecker sum),
//     X_a = diag(sqrt(mult_a)) L1_a diag(sqrt(mult_a)) / h_a^2,
// C = diag(c), L1 the 1-D Neumann path Laplacian, mult_a the per-axis sharing
// multiplicity.  M = -A + sI = C S C + sI is SPD; we solve it by conjugate
// gradients preconditioned with C^-1 (S + sigma I)^-1 C^-1, applied exactly by
// fast diagonalisation (17 x 17 eigenbases per axis), sigma = s/(c_min c_max):
// the preconditioned spectrum lies in [c_min/c_max, c_max/c_min] and clusters
// at 1, so 15-16 iterations reach |r| <= 1e-14 |b| (checked against SuperLU:
// 3e-15).  One CTA owns one right-hand side with every vector in shared
// memory, so the solve streams nothing from HBM.  Any orthonormal basis of the
// same Krylov space yields the same Lanczos chain (the QR gauges are fixed by
// positive diagonals), which is what makes CholQR2 a valid stand-in for the
// reference's pivoted Householder QR when no deflation occurs.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sfw_common.cuh"
#include "sfw_linalg.cuh"

namespace sfw {

constexpr int PMAX = 32;

// ---------------------------------------------------------------------------
// 1-D operator tables: per (axis, pattern) with pattern bit0 = low end shared,
// bit1 = high end shared.  X = D L1 D / h^2, D = diag(sqrt(mult)); cyclic
// Jacobi eigen-decomposition X = Q diag(lam) Q^T.
__global__ void k_axis_eig(int px, int py, int pz, double hx, double hy, double hz, double* Qt, double* lamt,
                           double* dt, double* et) {
    const int t = threadIdx.x;
    if (t >= 12) return;
    const int a = t / 4, pat = t % 4;
    const int n = a == 0 ? px : a == 1 ? py : pz;
    const double h = a == 0 ? hx : a == 1 ? hy : hz;
    double X[PMAX * PMAX], V[PMAX * PMAX], sm[PMAX];
    for (int i = 0; i < n; ++i) sm[i] = 1.0;
    if (pat & 1) sm[0] = sqrt(2.0);
    if (pat & 2) sm[n - 1] = sqrt(2.0);
    const double ih2 = 1.0 / (h * h);
    for (int i = 0; i < n * n; ++i) X[i] = 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        X[i * n + i] += sm[i] * sm[i] * ih2;
        X[(i + 1) * n + i + 1] += sm[i + 1] * sm[i + 1] * ih2;
        X[i * n + i + 1] -= sm[i] * sm[i + 1] * ih2;
        X[(i + 1) * n + i] -= sm[i] * sm[i + 1] * ih2;
    }
    double* d = dt + (a * 4 + pat) * PMAX;
    double* e = et + (a * 4 + pat) * PMAX;
    for (int i = 0; i < n; ++i) {
        d[i] = X[i * n + i];
        e[i] = (i + 1 < n) ? X[i * n + i + 1] : 0.0;
    }
    for (int i = 0; i < n * n; ++i) V[i] = (i / n == i % n) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int p = 0; p < n; ++p) {
            dia += X[p * n + p] * X[p * n + p];
            for (int q = p + 1; q < n; ++q) off += X[p * n + q] * X[p * n + q];
        }
        if (off <= 1e-32 * dia) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = X[p * n + q];
                if (apq == 0.0) continue;
                const double theta = (X[q * n + q] - X[p * n + p]) / (2.0 * apq);
                const double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
                for (int k = 0; k < n; ++k) {
                    const double xkp = X[k * n + p], xkq = X[k * n + q];
                    X[k * n + p] = c * xkp - s * xkq;
                    X[k * n + q] = s * xkp + c * xkq;
                }
                for (int k = 0; k < n; ++k) {
                    const double xpk = X[p * n + k], xqk = X[q * n + k];
                    X[p * n + k] = c * xpk - s * xqk;
                    X[q * n + k] = s * xpk + c * xqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V[k * n + p], vkq = V[k * n + q];
                    V[k * n + p] = c * vkp - s * vkq;
                    V[k * n + q] = s * vkp + c * vkq;
                }
            }
    }
    double* Q = Qt + (size_t)(a * 4 + pat) * PMAX * PMAX;
    double* lam = lamt + (a * 4 + pat) * PMAX;
    for (int i = 0; i < n * n; ++i) Q[i] = V[i];
    for (int i = 0; i < n; ++i) lam[i] = fmax(X[i * n + i], 0.0);
}

// ---------------------------------------------------------------------------
// face inputs F (rom.py:45-86) written into the first w columns of V.
__device__ __forceinline__ void face_window(const int* P, int f, int mask, int& ax, int& layer, int& a1, int& a2,
                                            int& lo1, int& hi1, int& lo2, int& hi2) {
    ax = f >> 1;
    layer = (f & 1) ? P[ax] - 1 : 0;
    const bool mine = (mask >> f) & 1;
    int lohi[3][2];
    for (int a = 0; a < 3; ++a) {
        int lo = 0, hi = P[a];
        if (a != ax) {
            for (int side = 0; side < 2; ++side) {
                const bool cross = (mask >> (2 * a + side)) & 1;
                const bool trim = (cross != mine) ? cross : (a < ax);
                if (trim) {
                    if (side == 0)
                        lo = 1;
                    else
                        hi = P[a] - 1;
                }
            }
        }
        lohi[a][0] = lo;
        lohi[a][1] = hi;
    }
    a1 = (ax == 0) ? 1 : 0;
    a2 = (ax == 2) ? 1 : 2;
    lo1 = lohi[a1][0];
    hi1 = lohi[a1][1];
    lo2 = lohi[a2][0];
    hi2 = lohi[a2][1];
}

__device__ __forceinline__ double dct_mode(int n, int i, int j) {
    // rom.py:45-52: cos(pi * ((i + 0.5) * j) / n) * (j == 0 ? sqrt(1/n) : sqrt(2/n))
    const double v = cos((M_PI * ((i + 0.5) * (double)j)) / n);
    return v * (j == 0 ? sqrt(1.0 / n) : sqrt(2.0 / n));
}

__global__ void k_face_basis(int px, int py, int pz, int m, int kk, const int* __restrict__ mask, double* V,
                             long long ldn, long long sV) {
    const int f = blockIdx.x, b = blockIdx.y;
    const int P[3] = {px, py, pz};
    int ax, layer, a1, a2, lo1, hi1, lo2, hi2;
    face_window(P, f, mask[b], ax, layer, a1, a2, lo1, hi1, lo2, hi2);
    const int na = hi1 - lo1, nb = hi2 - lo2;
    double* Vb = V + (size_t)b * sV;
    for (int idx = threadIdx.x; idx < na * nb * m; idx += blockDim.x) {
        const int row = idx / m, col = idx % m;
        const int ia = row / nb, ib = row % nb;
        const int al = col / kk, be = col % kk;
        int crd[3];
        crd[ax] = layer;
        crd[a1] = lo1 + ia;
        crd[a2] = lo2 + ib;
        const long long node = ((long long)crd[0] * py + crd[1]) * pz + crd[2];
        Vb[(size_t)(f * m + col) * ldn + node] = dct_mode(na, ia, al) * dct_mode(nb, ib, be);
    }
}

// ---------------------------------------------------------------------------
// PCG for M x = b, M = C S C + s I, preconditioner C^-1 (S + sigma)^-1 C^-1.
struct PcgArgs {
    int px, py, pz, N, ncols;
    long long ldn;
    double shift, tol;
    int maxit;
    const double* c;       // [B][N]
    const int* mask;       // [B]
    const double* Qt;      // [3][4][PMAX*PMAX]
    const double* lamt;    // [3][4][PMAX]
    const double* dt;      // [3][4][PMAX]
    const double* et;      // [3][4][PMAX]
    const double* rhs;     // column j of subdomain b at rhs + b*sR + j*ldn
    long long sR;
    double* out;           // writes -x
    long long sO;
    int* iters;            // [B*ncols]
};

template <int PT>
__device__ __forceinline__ void line_pass(double* z, const double* Q, int n, int nlines, int stride, int lstride_a,
                                          int lstride_b, int nb_inner, bool fwd) {
    // line l -> base = (l / nb_inner) * lstride_a + (l % nb_inner) * lstride_b
    // PT > 0: Q points at the direction-specific compact table Qd[i][k] (row stride QS = PT+1,
    //         16-B aligned rows) with y[k] = sum_i Qd[i][k] v[i]  -> 128-bit loads of Q pairs.
    // PT = 0: generic n <= PMAX, Q is the PMAX x PMAX table (forward Q[i][k], backward Q[k][i]).
    constexpr int PN = PT > 0 ? PT : PMAX;
    constexpr int QS = PT > 0 ? ((PT + 1) & ~1) : PMAX;
    for (int l = threadIdx.x; l < nlines; l += blockDim.x) {
        const int base = (l / nb_inner) * lstride_a + (l % nb_inner) * lstride_b;
        double v[PN], y[PN];
        if (PT > 0) {
#pragma unroll
            for (int i = 0; i < PN; ++i) v[i] = z[base + i * stride];
#pragma unroll
            for (int k = 0; k < PN; ++k) y[k] = 0.0;
#pragma unroll
            for (int i = 0; i < PN; ++i) {
                const double* qr = Q + i * QS;
#pragma unroll
                for (int k = 0; k + 1 < PN; k += 2) {
                    const double2 q = *reinterpret_cast<const double2*>(qr + k);
                    y[k] = fma(q.x, v[i], y[k]);
                    y[k + 1] = fma(q.y, v[i], y[k + 1]);
                }
                if (PN & 1) y[PN - 1] = fma(qr[PN - 1], v[i], y[PN - 1]);
            }
#pragma unroll
            for (int k = 0; k < PN; ++k) z[base + k * stride] = y[k];
        } else {
            for (int i = 0; i < n; ++i) v[i] = z[base + i * stride];
            for (int k = 0; k < n; ++k) {
                double s = 0.0;
                for (int i = 0; i < n; ++i) s = fma(fwd ? Q[i * n + k] : Q[k * n + i], v[i], s);
                y[k] = s;
            }
            for (int k = 0; k < n; ++k) z[base + k * stride] = y[k];
        }
    }
    __syncthreads();
}

template <int PT>
__global__ void __launch_bounds__(512, 1) k_pcg(const PcgArgs a) {
    extern __shared__ __align__(16) double sh[];
    const int N = a.N, px = PT > 0 ? PT : a.px, py = PT > 0 ? PT : a.py, pz = PT > 0 ? PT : a.pz;
    constexpr int QS = PT > 0 ? ((PT + 1) & ~1) : PMAX;        // compact row stride
    constexpr int QT = PT > 0 ? PT * QS : PMAX * PMAX;        // one table
    double* c = sh;
    double* ic = c + N;                // 1/c
    double* r = ic + N;
    double* p = r + N;
    double* z = p + N;
    double* Q = sh + ((5 * N + 1) & ~1);  // 16-B aligned;  PT > 0: [3 axes][fwd, bwd][PT][QS];  PT = 0: [3][PMAX*PMAX]
    double* lam = Q + (PT > 0 ? 6 : 3) * QT;
    double* dd = lam + 3 * PMAX;
    double* ee = dd + 3 * PMAX;
    double* red = ee + 3 * PMAX;       // 40
    const int b = blockIdx.x / a.ncols, j = blockIdx.x % a.ncols;
    const int mask = a.mask[b];
    const int P[3] = {px, py, pz};
    for (int ax = 0; ax < 3; ++ax) {
        const int pat = ((mask >> (2 * ax)) & 1) | (((mask >> (2 * ax + 1)) & 1) << 1);
        const int n = P[ax];
        const double* Qg = a.Qt + (size_t)(ax * 4 + pat) * PMAX * PMAX;  // compact n x n, row-major
        if (PT > 0) {
            for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
                const int i = idx / n, k = idx % n;
                Q[(2 * ax) * QT + i * QS + k] = Qg[idx];          // forward:  Qd[i][k] = Q[i][k]
                Q[(2 * ax + 1) * QT + k * QS + i] = Qg[idx];      // backward: Qd[i][k] = Q[k][i]
            }
        } else {
            for (int i = threadIdx.x; i < n * n; i += blockDim.x) Q[ax * QT + i] = Qg[i];
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            lam[ax * PMAX + i] = a.lamt[(ax * 4 + pat) * PMAX + i];
            dd[ax * PMAX + i] = a.dt[(ax * 4 + pat) * PMAX + i];
            ee[ax * PMAX + i] = a.et[(ax * 4 + pat) * PMAX + i];
        }
    }
    const double* cg = a.c + (size_t)b * N;
    const double* bg = a.rhs + (size_t)b * a.sR + (size_t)j * a.ldn;
    double* og = a.out + (size_t)b * a.sO + (size_t)j * a.ldn;  // accumulates -x
    double cmin = 1e308, cmax = 0.0, bb = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const double ci = cg[i];
        c[i] = ci;
        ic[i] = 1.0 / ci;
        cmin = fmin(cmin, ci);
        cmax = fmax(cmax, ci);
        const double bi = bg[i];
        r[i] = bi;
        og[i] = 0.0;
        bb = fma(bi, bi, bb);
    }
    cmax = block_max(cmax, red);
    cmin = -block_max(-cmin, red);
    bb = block_sum(bb, red);
    const double sigma = a.shift / (cmin * cmax);
    const double s = a.shift;
    const int sy = pz, sx = py * pz;
    auto Qf = [&](int ax) { return PT > 0 ? Q + (2 * ax) * QT : Q + ax * QT; };
    auto Qb = [&](int ax) { return PT > 0 ? Q + (2 * ax + 1) * QT : Q + ax * QT; };

    auto lpass = [&](const double* Qd, int n, int nl, int stride, int la, int lb, int nbi, bool fwd) {
        line_pass<PT>(z, Qd, n, nl, stride, la, lb, nbi, fwd);
    };
    auto precond = [&]() {  // z = P^-1 r
        for (int i = threadIdx.x; i < N; i += blockDim.x) z[i] = r[i] * ic[i];
        __syncthreads();
        lpass(Qf(0), px, py * pz, sx, 1, 1, py * pz, true);      // x lines: base = l
        lpass(Qf(1), py, px * pz, sy, sx, 1, pz, true);          // y lines
        lpass(Qf(2), pz, px * py, 1, pz, 0, 1, true);            // z lines: base = l*pz
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const int ix = i / sx, iy = (i / sy) % py, iz = i % pz;
            z[i] = z[i] * __drcp_rn(((lam[ix] + lam[PMAX + iy]) + lam[2 * PMAX + iz]) + sigma);
        }
        __syncthreads();
        lpass(Qb(2), pz, px * py, 1, pz, 0, 1, false);
        lpass(Qb(1), py, px * pz, sy, sx, 1, pz, false);
        lpass(Qb(0), px, py * pz, sx, 1, 1, py * pz, false);
        for (int i = threadIdx.x; i < N; i += blockDim.x) z[i] = z[i] * ic[i];
        __syncthreads();
    };

    precond();
    double rho = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        p[i] = z[i];
        rho = fma(r[i], z[i], rho);
    }
    rho = block_sum(rho, red);
    int it = 0, status = -1;
    const double tol2 = a.tol * a.tol * bb;
    if (bb == 0.0) status = 0;
    for (it = 0; status < 0 && it < a.maxit; ++it) {
        // q = M p = c .* S (c .* p) + s p  -> stored in z
        double pq = 0.0;
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const int ix = i / sx, iy = (i / sy) % py, iz = i % pz;
            const double ui = c[i] * p[i];
            double su = (dd[ix] + dd[PMAX + iy] + dd[2 * PMAX + iz]) * ui;
            if (ix + 1 < px) su = fma(ee[ix], c[i + sx] * p[i + sx], su);
            if (ix > 0) su = fma(ee[ix - 1], c[i - sx] * p[i - sx], su);
            if (iy + 1 < py) su = fma(ee[PMAX + iy], c[i + sy] * p[i + sy], su);
            if (iy > 0) su = fma(ee[PMAX + iy - 1], c[i - sy] * p[i - sy], su);
            if (iz + 1 < pz) su = fma(ee[2 * PMAX + iz], c[i + 1] * p[i + 1], su);
            if (iz > 0) su = fma(ee[2 * PMAX + iz - 1], c[i - 1] * p[i - 1], su);
            const double q = fma(c[i], su, s * p[i]);
            z[i] = q;
            pq = fma(p[i], q, pq);
        }
        pq = block_sum(pq, red);
        if (!(pq > 0.0)) {
            status = -2;  // not positive definite: shift too small
            break;
        }
        const double alpha = rho / pq;
        double rr = 0.0;
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            og[i] = fma(-alpha, p[i], og[i]);  // og = -x
            const double ri = fma(-alpha, z[i], r[i]);
            r[i] = ri;
            rr = fma(ri, ri, rr);
        }
        rr = block_sum(rr, red);
        if (rr <= tol2) {
            status = it + 1;
            break;
        }
        precond();
        double rz = 0.0;
        for (int i = threadIdx.x; i < N; i += blockDim.x) rz = fma(r[i], z[i], rz);
        rz = block_sum(rz, red);
        const double beta = rz / rho;
        rho = rz;
        for (int i = threadIdx.x; i < N; i += blockDim.x) p[i] = fma(beta, p[i], z[i]);
        __syncthreads();
    }
    if (threadIdx.x == 0) a.iters[blockIdx.x] = status;
}

// ---------------------------------------------------------------------------
// k_pcg2: the same preconditioned CG as k_pcg, two right-hand sides of one subdomain per CTA
// (P = 17 only).  The two solves share c, the eigenbases and every barrier: the line passes deal
// 2 x 289 lines over 12 warps (75% of the threads busy instead of 56%), the block reductions carry
// both dot products through one barrier (ping-pong scratch, 1 barrier instead of 3), and r and 1/c
// live in registers (13 nodes per thread), so p and z of both solves fit the 227 KB of shared
// memory.  A solve that has converged stops updating (its lines are skipped) while the other runs.
constexpr int PCG2_T = 384;
constexpr int PCG2_NPT = (17 * 17 * 17 + PCG2_T - 1) / PCG2_T;  // nodes per thread

__device__ __forceinline__ void block_sum2(double& v0, double& v1, double* red) {
    // fixed-order: warp butterfly, then every thread sums the warp partials in warp order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) {
        red[2 * warp] = v0;
        red[2 * warp + 1] = v1;
    }
    __syncthreads();
    double t0 = red[0], t1 = red[1];
    for (int i = 1; i < nw; ++i) {
        t0 += red[2 * i];
        t1 += red[2 * i + 1];
    }
    v0 = t0;
    v1 = t1;
}

__device__ __forceinline__ void line_pass2(double* z0, double* z1, const double* Q, int nlines, int stride,
                                           int lstride_a, int lstride_b, int nb_inner, bool act0, bool act1) {
    constexpr int PN = 17, QS = 18;
    for (int l = threadIdx.x; l < 2 * nlines; l += blockDim.x) {
        const int j = l >= nlines;
        if (j ? !act1 : !act0) continue;
        const int ll = j ? l - nlines : l;
        double* z = j ? z1 : z0;
        const int base = (ll / nb_inner) * lstride_a + (ll % nb_inner) * lstride_b;
        double v[PN], y[PN];
#pragma unroll
        for (int i = 0; i < PN; ++i) v[i] = z[base + i * stride];
#pragma unroll
        for (int k = 0; k < PN; ++k) y[k] = 0.0;
#pragma unroll
        for (int i = 0; i < PN; ++i) {
            const double* qr = Q + i * QS;
#pragma unroll
            for (int k = 0; k + 1 < PN; k += 2) {
                const double2 q = *reinterpret_cast<const double2*>(qr + k);
                y[k] = fma(q.x, v[i], y[k]);
                y[k + 1] = fma(q.y, v[i], y[k + 1]);
            }
            y[PN - 1] = fma(qr[PN - 1], v[i], y[PN - 1]);
        }
#pragma unroll
        for (int k = 0; k < PN; ++k) z[base + k * stride] = y[k];
    }
    __syncthreads();
}

// The same line pass as one GEMM per 8-line tile on the DMMA pipe: Y (17 x 8 lines) = Qd^T V, with
// Qd^T padded to 24 x 20 (3 row tiles x 5 k-steps of mma.m8n8k4.f64; its 15 A fragments live in
// registers for the pass) and 37 tiles of 8 lines per solve, dealt over the CTA's warps.  Each tile's
// lines are read into registers before its MMAs (warp-collective), then written back in place.
__device__ __forceinline__ void line_pass2_dmma(double* z0, double* z1, const double* Q, int nlines, int stride,
                                                int lstride_a, int lstride_b, int nb_inner, bool act0, bool act1) {
    constexpr int PN = 17, QS = 18;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int q = lane & 3, r = lane >> 2;
    double af[3][5];
#pragma unroll
    for (int I = 0; I < 3; ++I)
#pragma unroll
        for (int kap = 0; kap < 5; ++kap) {
            const int kout = 8 * I + r, i = 4 * kap + q;
            af[I][kap] = (kout < PN && i < PN) ? Q[i * QS + kout] : 0.0;  // A[kout][i] = Qd[i][kout]
        }
    const int ntile = (nlines + 7) / 8;
    for (int t = warp; t < 2 * ntile; t += nw) {
        const int j = t >= ntile;
        if (j ? !act1 : !act0) continue;
        double* z = j ? z1 : z0;
        const int n0 = (t - j * ntile) * 8;
        const int lb = n0 + r;  // this lane's B-fragment line
        const int base_b = (lb / nb_inner) * lstride_a + (lb % nb_inner) * lstride_b;
        double bf[5];
#pragma unroll
        for (int kap = 0; kap < 5; ++kap) {
            const int i = 4 * kap + q;
            bf[kap] = (lb < nlines && i < PN) ? z[base_b + i * stride] : 0.0;
        }
        double acc[3][2];
#pragma unroll
        for (int I = 0; I < 3; ++I) {
            acc[I][0] = acc[I][1] = 0.0;
#pragma unroll
            for (int kap = 0; kap < 5; ++kap) dmma8x8x4(acc[I], af[I][kap], bf[kap]);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int lo = n0 + 2 * q + e;  // output line of acc[.][e]
            if (lo >= nlines) continue;
            const int base_o = (lo / nb_inner) * lstride_a + (lo % nb_inner) * lstride_b;
#pragma unroll
            for (int I = 0; I < 3; ++I) {
                const int kout = 8 * I + r;
                if (kout < PN) z[base_o + kout * stride] = acc[I][e];
            }
        }
    }
    __syncthreads();
}

#ifndef SFW_PCG_DMMA
#define SFW_PCG_DMMA 1
#endif
#if SFW_PCG_DMMA
#define LP2 line_pass2_dmma
#else
#define LP2 line_pass2
#endif
__global__ void __launch_bounds__(PCG2_T, 1) k_pcg2(const PcgArgs a) {
    extern __shared__ __align__(16) double sh[];
    constexpr int PT = 17, QS = 18, QT = PT * QS, N = PT * PT * PT;
    constexpr int px = PT, py = PT, pz = PT;
    double* c = sh;
    double* p0 = c + N;
    double* p1 = p0 + N;
    double* z0 = p1 + N;
    double* z1 = z0 + N;
    double* Q = sh + ((5 * N + 1) & ~1);  // [3 axes][fwd, bwd][PT][QS]
    double* lam = Q + 6 * QT;
    double* dd = lam + 3 * PMAX;
    double* ee = dd + 3 * PMAX;
    double* red = ee + 3 * PMAX;  // 2 x 2 x 32 (ping-pong)
    const int ncp = (a.ncols + 1) / 2;
    const int b = blockIdx.x / ncp, j0 = 2 * (blockIdx.x % ncp);
    const bool two = j0 + 1 < a.ncols;
    const int mask = a.mask[b];
    for (int ax = 0; ax < 3; ++ax) {
        const int pat = ((mask >> (2 * ax)) & 1) | (((mask >> (2 * ax + 1)) & 1) << 1);
        const double* Qg = a.Qt + (size_t)(ax * 4 + pat) * PMAX * PMAX;
        for (int idx = threadIdx.x; idx < PT * PT; idx += blockDim.x) {
            const int i = idx / PT, k = idx % PT;
            Q[(2 * ax) * QT + i * QS + k] = Qg[idx];
            Q[(2 * ax + 1) * QT + k * QS + i] = Qg[idx];
        }
        for (int i = threadIdx.x; i < PT; i += blockDim.x) {
            lam[ax * PMAX + i] = a.lamt[(ax * 4 + pat) * PMAX + i];
            dd[ax * PMAX + i] = a.dt[(ax * 4 + pat) * PMAX + i];
            ee[ax * PMAX + i] = a.et[(ax * 4 + pat) * PMAX + i];
        }
    }
    const double* cg = a.c + (size_t)b * N;
    const double* bg0 = a.rhs + (size_t)b * a.sR + (size_t)j0 * a.ldn;
    const double* bg1 = bg0 + a.ldn;
    double* og0 = a.out + (size_t)b * a.sO + (size_t)j0 * a.ldn;  // accumulates -x
    double* og1 = og0 + a.ldn;
    double r0[PCG2_NPT], r1[PCG2_NPT], ic[PCG2_NPT];
    double cmin = 1e308, cmax = 0.0, bb0 = 0.0, bb1 = 0.0;
#pragma unroll
    for (int t = 0; t < PCG2_NPT; ++t) {
        const int i = threadIdx.x + t * PCG2_T;
        r0[t] = r1[t] = ic[t] = 0.0;
        if (i < N) {
            const double ci = cg[i];
            c[i] = ci;
            ic[t] = 1.0 / ci;
            cmin = fmin(cmin, ci);
            cmax = fmax(cmax, ci);
            r0[t] = bg0[i];
            og0[i] = 0.0;
            bb0 = fma(r0[t], r0[t], bb0);
            if (two) {
                r1[t] = bg1[i];
                og1[i] = 0.0;
                bb1 = fma(r1[t], r1[t], bb1);
            }
        }
    }
    cmax = block_max(cmax, red);
    cmin = -block_max(-cmin, red);
    int rb = 0;  // ping-pong reduction buffer
    block_sum2(bb0, bb1, red + 64 * rb);
    rb ^= 1;
    // (sigma = s <1/c^2>, which centres the constant mode, measured the same: 14.83 against 14.97 mean iterations)
    const double sigma = a.shift / (cmin * cmax);
    const double s = a.shift;
    constexpr int sy = pz, sx = py * pz;
    bool act0 = true, act1 = two;

    auto precond = [&]() {  // z_j = P^-1 r_j for the active solves
#pragma unroll
        for (int t = 0; t < PCG2_NPT; ++t) {
            const int i = threadIdx.x + t * PCG2_T;
            if (i < N) {
                if (act0) z0[i] = r0[t] * ic[t];
                if (act1) z1[i] = r1[t] * ic[t];
            }
        }
        __syncthreads();
        LP2(z0, z1, Q + 0 * QT, py * pz, sx, 1, 1, py * pz, act0, act1);
        LP2(z0, z1, Q + 2 * QT, px * pz, sy, sx, 1, pz, act0, act1);
        LP2(z0, z1, Q + 4 * QT, px * py, 1, pz, 0, 1, act0, act1);
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const int ix = i / sx, iy = (i / sy) % py, iz = i % pz;
            const double d = __drcp_rn(((lam[ix] + lam[PMAX + iy]) + lam[2 * PMAX + iz]) + sigma);
            if (act0) z0[i] = z0[i] * d;
            if (act1) z1[i] = z1[i] * d;
        }
        __syncthreads();
        LP2(z0, z1, Q + 5 * QT, px * py, 1, pz, 0, 1, act0, act1);
        LP2(z0, z1, Q + 3 * QT, px * pz, sy, sx, 1, pz, act0, act1);
        LP2(z0, z1, Q + 1 * QT, py * pz, sx, 1, 1, py * pz, act0, act1);
#pragma unroll
        for (int t = 0; t < PCG2_NPT; ++t) {
            const int i = threadIdx.x + t * PCG2_T;
            if (i < N) {
                if (act0) z0[i] = z0[i] * ic[t];
                if (act1) z1[i] = z1[i] * ic[t];
            }
        }
        __syncthreads();
    };

    precond();
    double rho0 = 0.0, rho1 = 0.0;
#pragma unroll
    for (int t = 0; t < PCG2_NPT; ++t) {
        const int i = threadIdx.x + t * PCG2_T;
        if (i < N) {
            p0[i] = z0[i];
            rho0 = fma(r0[t], z0[i], rho0);
            if (two) {
                p1[i] = z1[i];
                rho1 = fma(r1[t], z1[i], rho1);
            }
        }
    }
    block_sum2(rho0, rho1, red + 64 * rb);
    rb ^= 1;
    int st0 = -1, st1 = two ? -1 : 0;
    const double tol0 = a.tol * a.tol * bb0, tol1 = a.tol * a.tol * bb1;
    if (bb0 == 0.0) st0 = 0;
    if (bb1 == 0.0) st1 = 0;
    act0 = st0 < 0;
    act1 = st1 < 0;
    for (int it = 0; (act0 || act1) && it < a.maxit; ++it) {
        // q = M p = c .* S (c .* p) + s p  -> stored in z
        double pq0 = 0.0, pq1 = 0.0;
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const int ix = i / sx, iy = (i / sy) % py, iz = i % pz;
            const double dsum = dd[ix] + dd[PMAX + iy] + dd[2 * PMAX + iz];
            const double ci = c[i];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (j ? !act1 : !act0) continue;
                const double* p = j ? p1 : p0;
                const double ui = ci * p[i];
                double su = dsum * ui;
                if (ix + 1 < px) su = fma(ee[ix], c[i + sx] * p[i + sx], su);
                if (ix > 0) su = fma(ee[ix - 1], c[i - sx] * p[i - sx], su);
                if (iy + 1 < py) su = fma(ee[PMAX + iy], c[i + sy] * p[i + sy], su);
                if (iy > 0) su = fma(ee[PMAX + iy - 1], c[i - sy] * p[i - sy], su);
                if (iz + 1 < pz) su = fma(ee[2 * PMAX + iz], c[i + 1] * p[i + 1], su);
                if (iz > 0) su = fma(ee[2 * PMAX + iz - 1], c[i - 1] * p[i - 1], su);
                const double q = fma(ci, su, s * p[i]);
                if (j) {
                    z1[i] = q;
                    pq1 = fma(p[i], q, pq1);
                } else {
                    z0[i] = q;
                    pq0 = fma(p[i], q, pq0);
                }
            }
        }
        block_sum2(pq0, pq1, red + 64 * rb);
        rb ^= 1;
        if (act0 && !(pq0 > 0.0)) st0 = -2;  // not positive definite: shift too small
        if (act1 && !(pq1 > 0.0)) st1 = -2;
        if (st0 == -2 || st1 == -2) break;
        const double al0 = act0 ? rho0 / pq0 : 0.0, al1 = act1 ? rho1 / pq1 : 0.0;
        double rr0 = 0.0, rr1 = 0.0;
#pragma unroll
        for (int t = 0; t < PCG2_NPT; ++t) {
            const int i = threadIdx.x + t * PCG2_T;
            if (i < N) {
                if (act0) {
                    og0[i] = fma(-al0, p0[i], og0[i]);
                    r0[t] = fma(-al0, z0[i], r0[t]);
                    rr0 = fma(r0[t], r0[t], rr0);
                }
                if (act1) {
                    og1[i] = fma(-al1, p1[i], og1[i]);
                    r1[t] = fma(-al1, z1[i], r1[t]);
                    rr1 = fma(r1[t], r1[t], rr1);
                }
            }
        }
        block_sum2(rr0, rr1, red + 64 * rb);
        rb ^= 1;
        if (act0 && rr0 <= tol0) st0 = it + 1;
        if (act1 && rr1 <= tol1) st1 = it + 1;
        act0 = st0 < 0;
        act1 = st1 < 0;
        if (!act0 && !act1) break;
        __syncthreads();  // z (q) reads above are done before the preconditioner overwrites z
        precond();
        double rz0 = 0.0, rz1 = 0.0;
#pragma unroll
        for (int t = 0; t < PCG2_NPT; ++t) {
            const int i = threadIdx.x + t * PCG2_T;
            if (i < N) {
                if (act0) rz0 = fma(r0[t], z0[i], rz0);
                if (act1) rz1 = fma(r1[t], z1[i], rz1);
            }
        }
        block_sum2(rz0, rz1, red + 64 * rb);
        rb ^= 1;
        const double be0 = act0 ? rz0 / rho0 : 0.0, be1 = act1 ? rz1 / rho1 : 0.0;
        if (act0) rho0 = rz0;
        if (act1) rho1 = rz1;
#pragma unroll
        for (int t = 0; t < PCG2_NPT; ++t) {
            const int i = threadIdx.x + t * PCG2_T;
            if (i < N) {
                if (act0) p0[i] = fma(be0, p0[i], z0[i]);
                if (act1) p1[i] = fma(be1, p1[i], z1[i]);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.iters[(size_t)b * a.ncols + j0] = st0;
        if (two) a.iters[(size_t)b * a.ncols + j0 + 1] = st1;
    }
}

// ---------------------------------------------------------------------------
// Y[:, col] = A V[:, col] = -c .* S (c .* v)     (the grid.py operator as a stencil)
__global__ void k_stencil(int px, int py, int pz, int N, int ncols, const double* __restrict__ c,
                          const int* __restrict__ mask, const double* __restrict__ dt, const double* __restrict__ et,
                          const double* __restrict__ V, long long ldn, long long sV, int col0,
                          double* __restrict__ Y, long long sY) {
    const int b = blockIdx.y, col = blockIdx.x;
    const int mk = mask[b];
    const int pat0 = (mk & 1) | (((mk >> 1) & 1) << 1), pat1 = ((mk >> 2) & 1) | (((mk >> 3) & 1) << 1),
              pat2 = ((mk >> 4) & 1) | (((mk >> 5) & 1) << 1);
    const double* d0 = dt + (0 * 4 + pat0) * PMAX;
    const double* d1 = dt + (1 * 4 + pat1) * PMAX;
    const double* d2 = dt + (2 * 4 + pat2) * PMAX;
    const double* e0 = et + (0 * 4 + pat0) * PMAX;
    const double* e1 = et + (1 * 4 + pat1) * PMAX;
    const double* e2 = et + (2 * 4 + pat2) * PMAX;
    const double* cb = c + (size_t)b * N;
    const double* v = V + (size_t)b * sV + (size_t)(col0 + col) * ldn;
    double* y = Y + (size_t)b * sY + (size_t)col * ldn;
    const int sy = pz, sx = py * pz;
    for (int i = blockIdx.z * blockDim.x + threadIdx.x; i < N; i += gridDim.z * blockDim.x) {
        const int ix = i / sx, iy = (i / sy) % py, iz = i % pz;
        double su = (d0[ix] + d1[iy] + d2[iz]) * (cb[i] * v[i]);
        if (ix + 1 < px) su = fma(e0[ix], cb[i + sx] * v[i + sx], su);
        if (ix > 0) su = fma(e0[ix - 1], cb[i - sx] * v[i - sx], su);
        if (iy + 1 < py) su = fma(e1[iy], cb[i + sy] * v[i + sy], su);
        if (iy > 0) su = fma(e1[iy - 1], cb[i - sy] * v[i - sy], su);
        if (iz + 1 < pz) su = fma(e2[iz], cb[i + 1] * v[i + 1], su);
        if (iz > 0) su = fma(e2[iz - 1], cb[i - 1] * v[i - 1], su);
        y[i] = -cb[i] * su;
    }
}

// squared Frobenius norm of a (rows x cols) column-major block per subdomain
__global__ void k_fro2(const double* __restrict__ X, int rows, int cols, long long ld, long long sX,
                       double* __restrict__ out) {
    __shared__ double red[40];
    const double* Xb = X + (size_t)blockIdx.x * sX;
    double s = 0.0;
    for (int col = 0; col < cols; ++col)
        for (int i = threadIdx.x; i < rows; i += blockDim.x) {
            const double v = Xb[(size_t)col * ld + i];
            s = fma(v, v, s);
        }
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// CholQR step on Gram matrices G (w x w col-major, stride sG):
//   G = R^T R (R upper, positive diagonal); Rinv = R^-1 (col-major, for X <- X Rinv).
//   mode 0: Rkeep = R, dprod = diag(R)
//   mode 1: Rout = R Rkeep (row-major) = the total R of CholQR2, dprod *= diag(R)
// status[b] |= 1 if the Cholesky breaks down (rank-deficient block).
__global__ void k_cholqr(const double* __restrict__ G, long long sG, int w, double* __restrict__ Rinv,
                         double* __restrict__ Rkeep, double* __restrict__ Rout, long long sRout,
                         double* __restrict__ dprod, int mode, int* __restrict__ status) {
    extern __shared__ double sm[];
    double* A = sm;          // w*w row-major
    double* X = A + w * w;   // w*w row-major (inverse)
    __shared__ int bad;
    const int b = blockIdx.x;
    const double* Gb = G + (size_t)b * sG;
    if (threadIdx.x == 0) bad = 0;
    for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
        const int i = idx / w, j = idx % w;
        A[idx] = Gb[i + (size_t)j * w];
    }
    __syncthreads();
    for (int k = 0; k < w; ++k) {
        if (threadIdx.x == 0) {
            const double d = A[k * w + k];
            if (!(d > 0.0)) {
                bad = 1;
                A[k * w + k] = 1.0;
            } else {
                A[k * w + k] = sqrt(d);
            }
        }
        __syncthreads();
        const double rkk = A[k * w + k];
        for (int j = k + 1 + threadIdx.x; j < w; j += blockDim.x) A[k * w + j] /= rkk;
        __syncthreads();
        const int rem = w - k - 1;
        for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
            const int i = k + 1 + idx / rem, j = k + 1 + idx % rem;
            if (j >= i) A[i * w + j] = fma(-A[k * w + i], A[k * w + j], A[i * w + j]);
        }
        __syncthreads();
    }
    // upper-triangular inverse, one column per thread
    for (int j = threadIdx.x; j < w; j += blockDim.x) {
        for (int i = w - 1; i >= 0; --i) {
            if (i > j) {
                X[i * w + j] = 0.0;
                continue;
            }
            double s = (i == j) ? 1.0 : 0.0;
            for (int k = i + 1; k <= j; ++k) s = fma(-A[i * w + k], X[k * w + j], s);
            X[i * w + j] = s / A[i * w + i];
        }
    }
    __syncthreads();
    double* Ri = Rinv + (size_t)b * w * w;
    for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
        const int i = idx % w, j = idx / w;  // col-major write
        Ri[idx] = X[i * w + j];
    }
    double* Rk = Rkeep + (size_t)b * w * w;
    if (mode == 0) {
        for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
            const int i = idx / w, j = idx % w;
            Rk[idx] = (j >= i) ? A[idx] : 0.0;
        }
        for (int i = threadIdx.x; i < w; i += blockDim.x) dprod[(size_t)b * w + i] = A[i * w + i];
    } else {
        for (int i = threadIdx.x; i < w; i += blockDim.x) dprod[(size_t)b * w + i] *= A[i * w + i];
        if (Rout) {
            double* Ro = Rout + (size_t)b * sRout;
            for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
                const int i = idx / w, j = idx % w;
                double s = 0.0;
                for (int k = i; k <= j; ++k) s = fma(A[i * w + k], Rk[k * w + j], s);
                Ro[idx] = (j >= i) ? s : 0.0;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && bad) status[b] |= 1;
}

// row-major symmetric part: out = 0.5 (G + G^T), G col-major w x w
__global__ void k_symmetrize(const double* __restrict__ G, long long sG, int w, double* __restrict__ out,
                             long long sO) {
    const double* Gb = G + (size_t)blockIdx.x * sG;
    double* Ob = out + (size_t)blockIdx.x * sO;
    for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
        const int i = idx / w, j = idx % w;
        Ob[idx] = 0.5 * (Gb[i + (size_t)j * w] + Gb[j + (size_t)i * w]);
    }
}

// in-place symmetrisation of K x K col-major matrices (rom.py:181)
__global__ void k_symmetrize_inplace(double* __restrict__ A, long long sA, int K) {
    double* Ab = A + (size_t)blockIdx.y * sA;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)K * K;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx % K), j = (int)(idx / K);
        if (i < j) {
            const double v = 0.5 * (Ab[i + (size_t)j * K] + Ab[j + (size_t)i * K]);
            Ab[i + (size_t)j * K] = v;
            Ab[j + (size_t)i * K] = v;
        }
    }
}

// ---------------------------------------------------------------------------
// S-fraction recursion (rom.py:265-316), one CTA per subdomain, w x w in smem.
// Tdiag / Toff / Entry row-major.  status: 0 ok, 10+j = singular scale at layer
// j+1, 20+j = singular link at layer j+1, 30 = LU breakdown, 40 = hat_1 != I.
__global__ void k_sfraction(const double* __restrict__ Td, const double* __restrict__ To,
                            const double* __restrict__ En, int L, int Ls, int w, double* __restrict__ gam,
                            double* __restrict__ hat, double* __restrict__ scl, double* __restrict__ condv,
                            int* __restrict__ status) {
    extern __shared__ double sm[];
    const int ww = w * w;
    double* G = sm;
    double* LU = G + ww;
    double* Y = LU + ww;
    double* Gm = Y + ww;   // gamma
    double* Gp = Gm + ww;  // gamma_prev
    double* Wk = Gp + ww;  // workspace
    int* piv = reinterpret_cast<int*>(Wk + ww);
    __shared__ int flag;
    __shared__ double red[40];
    const int b = blockIdx.x;
    const double* Tb = Td + (size_t)b * Ls * ww;
    const double* Ob = To + (size_t)b * Ls * ww;  // B_{j+1} at Ob + j*ww (stride Ls*ww per subdomain)
    double* gb = gam + (size_t)b * Ls * ww;
    double* hb = hat + (size_t)b * Ls * ww;
    double* sb = scl + (size_t)b * Ls * ww;
    int st = 0;
    for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
        const int i = idx / w, j = idx % w;
        G[idx] = En[(size_t)b * ww + j * w + i];  // G_1 = B_1^T
        Gp[idx] = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < L; ++j) {
        // LU of G^T (used by the congruence below) also gives the condition check
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
            const int i = idx / w, k = idx % w;
            LU[idx] = G[k * w + i];
        }
        __syncthreads();
        const bool lu_ok = sm_lu(LU, piv, w, &flag);
        const double cg = lu_ok ? sm_cond2_check(G, LU, piv, Wk, Y, w, 1e12, red, &flag)
                                : __longlong_as_double(0x7ff0000000000000LL);
        if (threadIdx.x == 0) condv[(size_t)b * 2 * Ls + 2 * j] = cg;
        if (!(cg <= 1e12)) {
            st = 10 + j;
            break;
        }
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) sb[(size_t)j * ww + idx] = G[idx];
        sm_matmul(G, false, G, true, Wk, w);  // hat = G G^T
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) hb[(size_t)j * ww + idx] = Wk[idx];
        // congruence: y = solve(G^T, A_j); z = solve(G^T, y^T)^T; sym   (rom.py:265-269)
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) Y[idx] = Tb[(size_t)j * ww + idx];
        __syncthreads();
        sm_lu_solve(LU, piv, Y, w, w);
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
            const int i = idx / w, k = idx % w;
            Wk[idx] = Y[k * w + i];
        }
        __syncthreads();
        sm_lu_solve(LU, piv, Wk, w, w);  // Wk = solve(G^T, y^T) ; z = Wk^T
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
            const int i = idx / w, k = idx % w;
            const double zs = 0.5 * (Wk[k * w + i] + Wk[i * w + k]);  // sym(z), z = Wk^T
            Gm[idx] = -zs - Gp[idx];
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) gb[(size_t)j * ww + idx] = Gm[idx];
        if (j + 1 < L) {
            for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) Y[idx] = Gm[idx];
            __syncthreads();
            const bool gl_ok = sm_lu(Y, piv, w, &flag);
            const double cl = gl_ok ? sm_cond2_check(Gm, Y, piv, Wk, LU, w, 1e12, red, &flag)
                                    : __longlong_as_double(0x7ff0000000000000LL);
            if (threadIdx.x == 0) condv[(size_t)b * 2 * Ls + 2 * j + 1] = cl;
            if (!(cl <= 1e12)) {
                st = 20 + j;
                break;
            }
            // G_{j+1} = solve(G^T Gamma_j, B_{j+1}^T)
            sm_matmul(G, true, Gm, false, LU, w);
            if (!sm_lu(LU, piv, w, &flag)) {
                st = 30;
                break;
            }
            for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
                const int i = idx / w, k = idx % w;
                G[idx] = Ob[(size_t)j * ww + k * w + i];
            }
            __syncthreads();
            sm_lu_solve(LU, piv, G, w, w);
        }
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) Gp[idx] = Gm[idx];
        __syncthreads();
    }
    if (st == 0) {
        // |hat_1 - I|_F <= 1e-8   (rom.py:410-414)
        double s = 0.0;
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
            const double d = hb[idx] - ((idx / w == idx % w) ? 1.0 : 0.0);
            s = fma(d, d, s);
        }
        s = block_sum(s, red);
        if (!(sqrt(s) <= 1e-8)) st = 40;
    }
    if (threadIdx.x == 0) status[b] = st;
}

// rows of the node-space basis V Q: out[t][k] = sum_l V[b][l][row] Q[b][l][k]
__global__ void k_basis_rows(const double* __restrict__ V, long long ldn, long long sV, const double* __restrict__ Q,
                             long long sQ, int K, const int* __restrict__ rb, const int* __restrict__ rrow,
                             double* __restrict__ out) {
    const int t = blockIdx.x;
    const int b = rb[t], row = rrow[t];
    const double* Vb = V + (size_t)b * sV;
    const double* Qb = Q + (size_t)b * sQ;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        double s = 0.0;
        for (int l = 0; l < K; ++l) s = fma(Vb[(size_t)l * ldn + row], Qb[l + (size_t)k * K], s);
        out[(size_t)t * K + k] = s;
    }
}

// ---------------------------------------------------------------------------
// host orchestration

#ifndef SFW_DGEMM2
#define SFW_DGEMM2 1
#endif
static void gemm(cudaStream_t st, bool ta, int M, int N, int K, double alpha, const double* A, long long lda,
                 long long sA, const double* B, long long ldb, long long sB, double beta, double* C, long long ldc,
                 long long sC, int batch) {
    GemmArgs g{M, N, K, alpha, beta, A, lda, sA, B, ldb, sB, C, ldc, sC};
    dim3 grid((N + 63) / 64, (M + 63) / 64, batch);
    // the cp.async kernel needs 16-B aligned operands: even leading dimensions and batch strides
    const bool al = !(((uintptr_t)A | (uintptr_t)B) & 15) && !((lda | ldb | sA | sB) & 1) && SFW_DGEMM2;
    static bool attr = false;
    if (al && !attr) {
        cudaFuncSetAttribute(k_dgemm2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DG2_SMEM);
        cudaFuncSetAttribute(k_dgemm2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DG2_SMEM);
        attr = true;
    }
    if (al && ta)
        k_dgemm2<true><<<grid, 128, DG2_SMEM, st>>>(g);
    else if (al)
        k_dgemm2<false><<<grid, 128, DG2_SMEM, st>>>(g);
    else if (ta)
        k_dgemm<true><<<grid, 128, 0, st>>>(g);
    else
        k_dgemm<false><<<grid, 128, 0, st>>>(g);
}

}  // namespace sfw

using namespace sfw;

// sfw_rom_desc / sfw_rom_out: include/sfw_b200.h

namespace {
struct DevBuf {
    std::vector<void*> ptrs;
    ~DevBuf() {
        for (void* p : ptrs) cudaFree(p);
    }
    template <typename T>
    T* get(size_t n) {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
};
}  // namespace

// Face inputs F of one subdomain (reference rom.py:55-86 subdomain_inputs), the same k_face_basis
// the batched build uses: out[c * N + node] = column c of the N x 6m input matrix.
extern "C" int sfw_face_inputs(int px, int py, int pz, int m, int nbr_mask, double* out, char* errbuf, int errlen) {
    const int kk = (int)std::lround(std::sqrt((double)m));
    if (m < 1 || kk * kk != m) return fail(SFW_ECONFIG, "modes per face must be a perfect square", errbuf, errlen);
    const long long N = (long long)px * py * pz, w = 6LL * m;
    double* V = nullptr;
    int* dm = nullptr;
    SFW_CUDA_TRY(cudaMalloc(&V, (size_t)N * w * 8));
    SFW_CUDA_TRY(cudaMalloc(&dm, 4));
    cudaMemset(V, 0, (size_t)N * w * 8);
    sfw_h2d(dm, &nbr_mask, 4);
    k_face_basis<<<dim3(6, 1), 128>>>(px, py, pz, m, kk, dm, V, N, N * w);
    cudaError_t e = cudaMemcpy(out, V, (size_t)N * w * 8, cudaMemcpyDeviceToHost);
    cudaFree(V);
    cudaFree(dm);
    if (e != cudaSuccess) return fail(SFW_ECUDA, cudaGetErrorString(e), errbuf, errlen);
    return 0;
}

// Y = A X for n_sub subdomains with the build's own stencil (k_axis_eig tables + k_stencil):
// the operator the GPU pipeline factors, so a caller can check it against an explicit
// SubdomainOperator.matrix (reference grid.py:415-458) before trusting the build.
extern "C" int sfw_subdomain_apply(int n_sub, const int* p, const double* h, const double* c, const int* nbr_mask,
                                   int ncols, const double* X, double* Y, char* errbuf, int errlen) {
    if (n_sub <= 0 || ncols <= 0) return 0;
    const int px = p[0], py = p[1], pz = p[2];
    if (px < 4 || py < 4 || pz < 4 || px > PMAX || py > PMAX || pz > PMAX)
        return fail(SFW_ECONFIG, "nodes per subdomain axis must be in [4, 32]", errbuf, errlen);
    const int N = px * py * pz;
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
        return fail(SFW_ECUDA, "stream creation failed", errbuf, errlen);
    int rc = 0;
    {
        DevBuf db;
        double* dQt = db.get<double>(12 * PMAX * PMAX);
        double* dlam = db.get<double>(12 * PMAX);
        double* ddt = db.get<double>(12 * PMAX);
        double* det = db.get<double>(12 * PMAX);
        double* dc = db.get<double>((size_t)n_sub * N);
        int* dm = db.get<int>(n_sub);
        double* dX = db.get<double>((size_t)n_sub * ncols * N);
        double* dY = db.get<double>((size_t)n_sub * ncols * N);
        if (!dQt || !dc || !dm || !dX || !dY) {
            rc = fail(SFW_ECUDA, "out of device memory in sfw_subdomain_apply", errbuf, errlen);
        } else {
            sfw_h2d(dc, c, (size_t)n_sub * N * 8);
            sfw_h2d(dm, nbr_mask, (size_t)n_sub * sizeof(int));
            sfw_h2d(dX, X, (size_t)n_sub * ncols * N * 8);
            k_axis_eig<<<1, 32, 0, st>>>(px, py, pz, h[0], h[1], h[2], dQt, dlam, ddt, det);
            k_stencil<<<dim3(ncols, n_sub, 8), 128, 0, st>>>(px, py, pz, N, ncols, dc, dm, ddt, det, dX, N,
                                                              (long long)ncols * N, 0, dY, (long long)ncols * N);
            cudaMemcpyAsync(Y, dY, (size_t)n_sub * ncols * N * 8, cudaMemcpyDeviceToHost, st);
            cudaError_t e = cudaStreamSynchronize(st);
            if (e == cudaSuccess) e = cudaGetLastError();
            if (e != cudaSuccess) rc = fail(SFW_ECUDA, cudaGetErrorString(e), errbuf, errlen);
        }
    }
    cudaStreamDestroy(st);
    return rc;
}

extern "C" int sfw_rom_build(const sfw_rom_desc* d, sfw_rom_out* o, char* errbuf, int errlen) {
    using clk = std::chrono::steady_clock;
    const int nsub = d->n_sub, m = d->m, n = d->n;
    const int w = 6 * m, L = n + 1, K = L * w;
    const int px = d->p[0], py = d->p[1], pz = d->p[2];
    const int N = px * py * pz;
    const long long ldn = (N + 7) & ~7LL;
    if (nsub <= 0) return 0;
    if ((size_t)6 * w * w * 8 + 1024 > 227 * 1024)
        return fail(SFW_ECONFIG, "the batched GPU build supports w = 6m <= 66 (m <= 11)", errbuf, errlen);
    if (px < 4 || py < 4 || pz < 4 || px > PMAX || py > PMAX || pz > PMAX)
        return fail(SFW_ECONFIG, "nodes per subdomain axis must be in [4, 32] for the GPU build", errbuf, errlen);
    const int kk = (int)std::lround(std::sqrt((double)m));
    if (kk * kk != m) return fail(SFW_ECONFIG, "modes per face must be a perfect square, got " + std::to_string(m), errbuf, errlen);
    if (!(d->shift > 0.0)) {
        const double hint = d->shift > 0 ? d->shift * 10.0 : 1e-8;
        char msg[256];
        snprintf(msg, sizeof msg,
                 "factorization of the shifted operator failed (-A + sI is not positive definite); the shift "
                 "%.3e is too small, try %.3e",
                 d->shift, hint);
        return fail(SFW_ENUMERICAL, msg, errbuf, errlen);
    }
    const bool p17 = (px == 17 && py == 17 && pz == 17);
    const size_t pcg_smem = p17 ? (size_t)(5 * N + 1 + 6 * 17 * 18 + 9 * PMAX + 40) * 8
                                : (size_t)(5 * N + 1 + 3 * PMAX * PMAX + 9 * PMAX + 40) * 8;
    if (pcg_smem > 227 * 1024)
        return fail(SFW_ECONFIG, "subdomain too large for the shared-memory PCG (N <= ~5100 nodes)", errbuf, errlen);

    // batch size from free memory
    size_t freeb = 0, totb = 0;
    cudaMemGetInfo(&freeb, &totb);
    const double per_sub = 8.0 * ((double)K * ldn + 2.0 * w * ldn + 3.0 * K * K + 4.0 * K * w + 8.0 * L * w * w + N);
    int B = d->batch > 0 ? d->batch : (int)std::max(1.0, std::min((double)nsub, 0.45 * freeb / per_sub));
    B = std::min(B, nsub);
    B = std::min(B, 65535);

    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    DevBuf db;
    double* dQt = db.get<double>(12 * PMAX * PMAX);
    double* dlam = db.get<double>(12 * PMAX);
    double* ddt = db.get<double>(12 * PMAX);
    double* det = db.get<double>(12 * PMAX);
    double* dc = db.get<double>((size_t)B * N);
    int* dmask = db.get<int>(B);
    double* V = db.get<double>((size_t)B * K * ldn);
    double* X = db.get<double>((size_t)B * w * ldn);
    double* Y = db.get<double>((size_t)B * K * w);
    double* Gm = db.get<double>((size_t)B * w * w);
    double* Ri = db.get<double>((size_t)B * w * w);
    double* Rk = db.get<double>((size_t)B * w * w);
    double* dpr = db.get<double>((size_t)B * w);
    double* fro = db.get<double>(B);
    int* it = db.get<int>((size_t)B * w);
    int* dstat = db.get<int>(B);
    int* sstat = db.get<int>(B);
    double* At = db.get<double>((size_t)B * K * K);
    double* Qz = db.get<double>((size_t)B * K * K);
    double* Ft = db.get<double>((size_t)B * K * w);
    double* Z = db.get<double>((size_t)B * K * w);
    double* Td = db.get<double>((size_t)B * L * w * w);
    double* To = db.get<double>((size_t)B * L * w * w);
    double* En = db.get<double>((size_t)B * w * w);
    double* Ga = db.get<double>((size_t)B * L * w * w);
    double* Ha = db.get<double>((size_t)B * L * w * w);
    double* Sc = db.get<double>((size_t)B * L * w * w);
    double* cnd = db.get<double>((size_t)B * 2 * L);
    int* drb = db.get<int>(std::max(1, d->n_rows));
    int* drr = db.get<int>(std::max(1, d->n_rows));
    double* drows = db.get<double>((size_t)std::max(1, d->n_rows) * K);
    double* dfull = d->full_basis ? db.get<double>((size_t)B * K * ldn) : nullptr;
    if (!dQt || !V || !At || !Qz || !Ga || !drows || (d->full_basis && !dfull)) {
        cudaStreamDestroy(st);
        return fail(SFW_ECUDA, "out of device memory for the ROM build batch", errbuf, errlen);
    }
    k_axis_eig<<<1, 32, 0, st>>>(px, py, pz, d->h[0], d->h[1], d->h[2], dQt, dlam, ddt, det);

    double t_solve = 0, t_orth = 0, t_proj = 0, t_lanc = 0, t_sfr = 0;
    int max_it = 0;
    long long sum_it = 0, n_it = 0;  // SFW_PCG_STATS: mean iteration count of the shifted solves
    std::vector<int> hit((size_t)B * w), hstat(B), hs2(B);
    std::vector<double> hfro(B), hdpr((size_t)B * w);
    const size_t ww = (size_t)w * w;
    std::vector<std::string> errors;
    int rc = 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto tmark = [&](double& acc, cudaEvent_t a, cudaEvent_t b) {
        float ms = 0;
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        acc += ms * 1e-3;
    };
    PcgArgs pa{};
    pa.px = px;
    pa.py = py;
    pa.pz = pz;
    pa.N = N;
    pa.ncols = w;
    pa.ldn = ldn;
    pa.shift = d->shift;
    pa.tol = 1e-14;
    pa.maxit = 1000;
    pa.c = dc;
    pa.mask = dmask;
    pa.Qt = dQt;
    pa.lamt = dlam;
    pa.dt = ddt;
    pa.et = det;
    pa.iters = it;
    const void* pcg_fn = p17 ? (const void*)k_pcg<17> : (const void*)k_pcg<0>;
    // P = 17: two right-hand sides per CTA (k_pcg2); SFW_PCG1 selects the one-RHS kernel
    const bool pcg2 = p17 && !getenv("SFW_PCG1");
    const size_t pcg2_smem = (size_t)(((5 * 4913 + 1) & ~1) + 6 * 17 * 18 + 9 * PMAX + 128) * 8;
    if (pcg2) cudaFuncSetAttribute(k_pcg2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pcg2_smem);
    cudaFuncSetAttribute(pcg_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pcg_smem);
    const size_t cq_smem = 2 * ww * 8;
    cudaFuncSetAttribute(k_cholqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cq_smem);
    const size_t sf_smem = 6 * ww * 8 + w * sizeof(int) + 16;
    cudaFuncSetAttribute(k_sfraction, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf_smem);


    const auto t_begin = clk::now();
    for (int i0 = 0; i0 < nsub && rc == 0; i0 += B) {
        const int nb = std::min(B, nsub - i0);
        cudaMemcpyAsync(dc, d->c + (size_t)i0 * N, (size_t)nb * N * 8, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dmask, d->nbr_mask + i0, nb * 4, cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(V, 0, (size_t)nb * K * ldn * 8, st);
        cudaMemsetAsync(dstat, 0, nb * 4, st);
        std::vector<int> keep(nb, L);
        k_face_basis<<<dim3(6, nb), 128, 0, st>>>(px, py, pz, m, kk, dmask, V, ldn, (long long)K * ldn);

        // ---------------- shifted-inverse Krylov rounds -----------------------
        for (int r = 1; r <= n; ++r) {
            cudaEventRecord(e0, st);
            pa.rhs = V + (size_t)(r - 1) * w * ldn;
            pa.sR = (long long)K * ldn;
            pa.out = X;
            pa.sO = (long long)w * ldn;
            if (pcg2)
                k_pcg2<<<nb * ((w + 1) / 2), PCG2_T, pcg2_smem, st>>>(pa);
            else if (p17)
                k_pcg<17><<<nb * w, 512, pcg_smem, st>>>(pa);
            else
                k_pcg<0><<<nb * w, 512, pcg_smem, st>>>(pa);
            cudaEventRecord(e1, st);
            tmark(t_solve, e0, e1);
            cudaMemcpy(hit.data(), it, (size_t)nb * w * 4, cudaMemcpyDeviceToHost);
            for (int b = 0; b < nb; ++b)
                for (int j = 0; j < w; ++j) {
                    const int v = hit[(size_t)b * w + j];
                    if (v < 0 && keep[b] == L) {
                        errors.push_back("subdomain " + std::to_string(i0 + b) +
                                         (v == -2 ? ": factorization of the shifted operator failed (not positive "
                                                    "definite); the shift is too small"
                                                  : ": shifted solve did not converge"));
                        keep[b] = -1;
                    }
                    max_it = std::max(max_it, v);
                    if (v > 0) {
                        sum_it += v;
                        ++n_it;
                    }
                }
            cudaEventRecord(e0, st);
            const int Kr = r * w;
            k_fro2<<<nb, 256, 0, st>>>(X, N, w, ldn, (long long)w * ldn, fro);
            for (int pass = 0; pass < 2; ++pass) {  // CGS2 (rom.py:125-127)
                gemm(st, true, Kr, w, N, 1.0, V, ldn, (long long)K * ldn, X, ldn, (long long)w * ldn, 0.0, Y, Kr,
                     (long long)K * w, nb);
                gemm(st, false, N, w, Kr, -1.0, V, ldn, (long long)K * ldn, Y, Kr, (long long)K * w, 1.0, X, ldn,
                     (long long)w * ldn, nb);
            }
            // CholQR2 -> block r of V
            double* Vr = V + (size_t)r * w * ldn;
            gemm(st, true, w, w, N, 1.0, X, ldn, (long long)w * ldn, X, ldn, (long long)w * ldn, 0.0, Gm, w, ww, nb);
            k_cholqr<<<nb, 128, cq_smem, st>>>(Gm, ww, w, Ri, Rk, nullptr, 0, dpr, 0, dstat);
            gemm(st, false, N, w, w, 1.0, X, ldn, (long long)w * ldn, Ri, w, ww, 0.0, Vr, ldn, (long long)K * ldn, nb);
            gemm(st, true, w, w, N, 1.0, Vr, ldn, (long long)K * ldn, Vr, ldn, (long long)K * ldn, 0.0, Gm, w, ww, nb);
            k_cholqr<<<nb, 128, cq_smem, st>>>(Gm, ww, w, Ri, Rk, nullptr, 0, dpr, 1, dstat);
            gemm(st, false, N, w, w, 1.0, Vr, ldn, (long long)K * ldn, Ri, w, ww, 0.0, X, ldn, (long long)w * ldn, nb);
            cudaMemcpy2DAsync(Vr, (size_t)K * ldn * 8, X, (size_t)w * ldn * 8, (size_t)w * ldn * 8, nb,
                              cudaMemcpyDeviceToDevice, st);
            cudaEventRecord(e1, st);
            tmark(t_orth, e0, e1);
            // deflation check (rom.py:128-136): |R_ii| > 1e-12 |raw|_F
            cudaMemcpy(hfro.data(), fro, nb * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(hdpr.data(), dpr, (size_t)nb * w * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(hstat.data(), dstat, nb * 4, cudaMemcpyDeviceToHost);
            if (const char* dump = getenv("SFW_ROM_DUMP")) {  // debug: V after this round, raw X
                cudaStreamSynchronize(st);
                std::vector<double> hv((size_t)nb * K * ldn);
                cudaMemcpy(hv.data(), V, hv.size() * 8, cudaMemcpyDeviceToHost);
                FILE* fp = fopen((std::string(dump) + "_V" + std::to_string(r) + ".bin").c_str(), "wb");
                if (fp) {
                    fwrite(hv.data(), 8, hv.size(), fp);
                    fclose(fp);
                }
            }
            if (getenv("SFW_ROM_DEBUG")) {
                for (int b = 0; b < std::min(nb, 2); ++b) {
                    fprintf(stderr, "[rom] round %d sub %d |raw| %.6e stat %d its %d R_ii:", r, i0 + b,
                            std::sqrt(hfro[b]), hstat[b], hit[(size_t)b * w]);
                    for (int i = 0; i < w; ++i) fprintf(stderr, " %.3e", hdpr[(size_t)b * w + i]);
                    fprintf(stderr, "\n");
                }
            }
            for (int b = 0; b < nb; ++b) {
                if (keep[b] != L) continue;
                const double tol = 1e-12 * std::max(std::sqrt(hfro[b]), 1e-300);
                bool full = (hstat[b] & 1) == 0;
                for (int i = 0; i < w && full; ++i) full = std::fabs(hdpr[(size_t)b * w + i]) > tol;
                if (!full) keep[b] = r;
            }
            cudaMemsetAsync(dstat, 0, nb * 4, st);
        }
        for (int b = 0; b < nb; ++b)
            if (keep[b] >= 0 && keep[b] < 2)
                errors.push_back("subdomain " + std::to_string(i0 + b) +
                                 ": shifted-inverse images of the face inputs are dependent already at depth 1; "
                                 "reduce the number of face modes");
        if (!errors.empty()) {
            rc = SFW_ENUMERICAL;
            break;
        }

        // Projection + Lanczos + S-fraction + outputs for subdomains [bo, bo+nbr) of this
        // batch, all with Lg complete layers (rom.py:375-395 truncation to complete blocks).
        auto finish = [&](int bo, int nbr, int Lg) {
            const int Kg = Lg * w;
            const double* Vb = V + (size_t)bo * K * ldn;
            const double* dcb = dc + (size_t)bo * N;
            const int* dmb = dmask + bo;
            const long long sV = (long long)K * ldn, sKK = (long long)K * K, sKw = (long long)K * w,
                            sL = (long long)L * ww, sX = (long long)w * ldn;
            // ---- Galerkin projection (rom.py:177-182)
            cudaEventRecord(e0, st);
            for (int c0 = 0; c0 < Kg; c0 += w) {
                k_stencil<<<dim3(w, nbr, 8), 128, 0, st>>>(px, py, pz, N, w, dcb, dmb, ddt, det, Vb, ldn, sV, c0, X,
                                                           sX);
                gemm(st, true, Kg, w, N, 1.0, Vb, ldn, sV, X, ldn, sX, 0.0, At + (size_t)c0 * Kg, Kg, sKK, nbr);
            }
            k_symmetrize_inplace<<<dim3(64, nbr), 256, 0, st>>>(At, sKK, Kg);
            gemm(st, true, Kg, w, N, 1.0, Vb, ldn, sV, Vb, ldn, sV, 0.0, Ft, Kg, sKw, nbr);
            cudaEventRecord(e1, st);
            tmark(t_proj, e0, e1);
            // ---- block Lanczos (rom.py:202-262)
            cudaEventRecord(e0, st);
            k_fro2<<<nbr, 256, 0, st>>>(At, Kg, Kg, Kg, sKK, fro);
            gemm(st, true, w, w, Kg, 1.0, Ft, Kg, sKw, Ft, Kg, sKw, 0.0, Gm, w, ww, nbr);
            k_cholqr<<<nbr, 128, cq_smem, st>>>(Gm, ww, w, Ri, Rk, nullptr, 0, dpr, 0, dstat);
            gemm(st, false, Kg, w, w, 1.0, Ft, Kg, sKw, Ri, w, ww, 0.0, Z, Kg, sKw, nbr);
            gemm(st, true, w, w, Kg, 1.0, Z, Kg, sKw, Z, Kg, sKw, 0.0, Gm, w, ww, nbr);
            k_cholqr<<<nbr, 128, cq_smem, st>>>(Gm, ww, w, Ri, Rk, En, ww, dpr, 1, dstat);
            gemm(st, false, Kg, w, w, 1.0, Z, Kg, sKw, Ri, w, ww, 0.0, Qz, Kg, sKK, nbr);
            cudaStreamSynchronize(st);
            cudaMemcpy(hfro.data(), fro, nbr * 8, cudaMemcpyDeviceToHost);
            std::vector<int> lost(nbr, 0);
            for (int j = 0; j < Lg; ++j) {
                const double* Qj = Qz + (size_t)j * w * Kg;
                gemm(st, false, Kg, w, Kg, 1.0, At, Kg, sKK, Qj, Kg, sKK, 0.0, Z, Kg, sKw, nbr);
                if (j > 0)  // Z -= Q_{j-1} B_j^T  (row-major B read as column-major = B^T)
                    gemm(st, false, Kg, w, w, -1.0, Qj - (size_t)w * Kg, Kg, sKK, To + (size_t)(j - 1) * ww, w, sL,
                         1.0, Z, Kg, sKw, nbr);
                gemm(st, true, w, w, Kg, 1.0, Qj, Kg, sKK, Z, Kg, sKw, 0.0, Gm, w, ww, nbr);
                k_symmetrize<<<nbr, 256, 0, st>>>(Gm, ww, w, Td + (size_t)j * ww, sL);
                if (j + 1 == Lg) break;
                gemm(st, false, Kg, w, w, -1.0, Qj, Kg, sKK, Td + (size_t)j * ww, w, sL, 1.0, Z, Kg, sKw, nbr);
                const int jb = (j + 1) * w;
                for (int pass = 0; pass < 2; ++pass) {
                    gemm(st, true, jb, w, Kg, 1.0, Qz, Kg, sKK, Z, Kg, sKw, 0.0, Y, jb, sKw, nbr);
                    gemm(st, false, Kg, w, jb, -1.0, Qz, Kg, sKK, Y, jb, sKw, 1.0, Z, Kg, sKw, nbr);
                }
                double* Qn = Qz + (size_t)(j + 1) * w * Kg;
                gemm(st, true, w, w, Kg, 1.0, Z, Kg, sKw, Z, Kg, sKw, 0.0, Gm, w, ww, nbr);
                k_cholqr<<<nbr, 128, cq_smem, st>>>(Gm, ww, w, Ri, Rk, nullptr, 0, dpr, 0, dstat);
                gemm(st, false, Kg, w, w, 1.0, Z, Kg, sKw, Ri, w, ww, 0.0, Qn, Kg, sKK, nbr);
                gemm(st, true, w, w, Kg, 1.0, Qn, Kg, sKK, Qn, Kg, sKK, 0.0, Gm, w, ww, nbr);
                k_cholqr<<<nbr, 128, cq_smem, st>>>(Gm, ww, w, Ri, Rk, To + (size_t)j * ww, sL, dpr, 1, dstat);
                gemm(st, false, Kg, w, w, 1.0, Qn, Kg, sKK, Ri, w, ww, 0.0, Z, Kg, sKw, nbr);
                cudaMemcpy2DAsync(Qn, (size_t)sKK * 8, Z, (size_t)sKw * 8, (size_t)Kg * w * 8, nbr,
                                  cudaMemcpyDeviceToDevice, st);
                // rank check (rom.py:239-245): |diag B_{j+1}| > 1e-11 |A~|_F / sqrt(K)
                cudaStreamSynchronize(st);
                cudaMemcpy(hdpr.data(), dpr, (size_t)nbr * w * 8, cudaMemcpyDeviceToHost);
                cudaMemcpy(hstat.data(), dstat, nbr * 4, cudaMemcpyDeviceToHost);
                for (int b = 0; b < nbr; ++b) {
                    const double tol = 1e-11 * std::max(std::sqrt(hfro[b]) / std::sqrt((double)Kg), 1e-300);
                    bool full = (hstat[b] & 1) == 0;
                    for (int i = 0; i < w && full; ++i) full = std::fabs(hdpr[(size_t)b * w + i]) > tol;
                    if (!full) lost[b] = 1;
                }
                cudaMemsetAsync(dstat, 0, nbr * 4, st);
            }
            cudaEventRecord(e1, st);
            tmark(t_lanc, e0, e1);
            bool bad = false;
            for (int b = 0; b < nbr; ++b)
                if (lost[b]) {
                    errors.push_back("subdomain " + std::to_string(i0 + bo + b) +
                                     ": tridiagonalization lost rank; try a different expansion shift");
                    bad = true;
                }
            if (bad) return;
            // ---- S-fraction (rom.py:265-316)
            cudaEventRecord(e0, st);
            k_sfraction<<<nbr, 256, sf_smem, st>>>(Td, To, En, Lg, L, w, Ga, Ha, Sc, cnd, sstat);
            cudaEventRecord(e1, st);
            tmark(t_sfr, e0, e1);
            cudaMemcpy(hs2.data(), sstat, nbr * 4, cudaMemcpyDeviceToHost);
            for (int b = 0; b < nbr; ++b) {
                const int s2 = hs2[b];
                if (s2 == 0) continue;
                std::string msg;
                if (s2 >= 10 && s2 < 20)
                    msg = "chain scale matrix at layer " + std::to_string(s2 - 9) +
                          " is numerically singular (condition > 1e+12); the reduction basis is unusable at this "
                          "size, reduce the layer count";
                else if (s2 >= 20 && s2 < 30)
                    msg = "chain link matrix at layer " + std::to_string(s2 - 19) +
                          " is numerically singular (condition > 1e+12); reduce the layer count";
                else if (s2 == 40)
                    msg = "first inverse-mass block deviates from identity; the input block was not kept verbatim";
                else
                    msg = "singular matrix in the S-fraction recursion";
                errors.push_back("subdomain " + std::to_string(i0 + bo + b) + ": " + msg);
                bad = true;
            }
            if (bad) return;
            // ---- outputs
            const int g0 = i0 + bo;
            const cudaMemcpyKind kind = d->out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
            const size_t lp = (size_t)L * ww * 8, lw = (size_t)Lg * ww * 8;
            cudaMemcpy2DAsync(o->gammas + (size_t)g0 * L * ww, lp, Ga, lp, lw, nbr, kind, st);
            cudaMemcpy2DAsync(o->gamma_hats + (size_t)g0 * L * ww, lp, Ha, lp, lw, nbr, kind, st);
            cudaMemcpy2DAsync(o->scales + (size_t)g0 * L * ww, lp, Sc, lp, lw, nbr, kind, st);
            if (o->tdiag) cudaMemcpy2DAsync(o->tdiag + (size_t)g0 * L * ww, lp, Td, lp, lw, nbr, cudaMemcpyDeviceToHost, st);
            if (o->toff && Lg > 1)
                cudaMemcpy2DAsync(o->toff + (size_t)g0 * (L - 1) * ww, (size_t)(L - 1) * ww * 8, To, lp,
                                  (size_t)(Lg - 1) * ww * 8, nbr, cudaMemcpyDeviceToHost, st);
            std::vector<int> rb, rr, ri;
            for (int t = 0; t < d->n_rows; ++t) {
                const int sidx = d->row_sub[t];
                if (sidx >= g0 && sidx < g0 + nbr) {
                    rb.push_back(sidx - g0);
                    rr.push_back(d->row_node[t]);
                    ri.push_back(t);
                }
            }
            if (!rb.empty() && o->basis_rows) {
                cudaMemcpyAsync(drb, rb.data(), rb.size() * 4, cudaMemcpyHostToDevice, st);
                cudaMemcpyAsync(drr, rr.data(), rr.size() * 4, cudaMemcpyHostToDevice, st);
                k_basis_rows<<<(unsigned)rb.size(), 128, 0, st>>>(Vb, ldn, sV, Qz, sKK, Kg, drb, drr, drows);
                std::vector<double> hrows(rb.size() * Kg);
                cudaMemcpyAsync(hrows.data(), drows, hrows.size() * 8, cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                for (size_t q = 0; q < ri.size(); ++q)
                    std::memcpy(o->basis_rows + (size_t)ri[q] * K, hrows.data() + q * Kg, (size_t)Kg * 8);
            }
            if (d->full_basis && o->basis) {
                gemm(st, false, N, Kg, Kg, 1.0, Vb, ldn, sV, Qz, Kg, sKK, 0.0, dfull, ldn, sV, nbr);
                for (int t = 0; t < nbr; ++t)
                    cudaMemcpy2DAsync(o->basis + (size_t)(g0 + t) * K * N, (size_t)N * 8, dfull + (size_t)t * sV,
                                      (size_t)ldn * 8, (size_t)N * 8, (size_t)Kg, cudaMemcpyDeviceToHost, st);
            }
            cudaStreamSynchronize(st);
            for (int t = 0; t < nbr; ++t) {
                o->layers[g0 + t] = Lg;
                o->flags[g0 + t] = (Lg < L) ? 3 : 0;
                if (o->status) o->status[g0 + t] = 0;
            }
        };
        bool uniform = true;
        for (int b = 0; b < nb; ++b) uniform = uniform && keep[b] == L;
        if (uniform) {
            finish(0, nb, L);
        } else {
            for (int b = 0; b < nb && errors.empty(); ++b) finish(b, 1, keep[b]);
        }
        if (!errors.empty()) {
            rc = SFW_ENUMERICAL;
            break;
        }
    }
    cudaError_t ce = cudaStreamSynchronize(st);
    if (ce == cudaSuccess) ce = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    if (o->stats) {
        o->stats[0] = t_solve;
        o->stats[1] = t_orth;
        o->stats[2] = t_proj;
        o->stats[3] = t_lanc;
        o->stats[4] = t_sfr;
        o->stats[5] = max_it;
        if (getenv("SFW_PCG_STATS") && n_it)
            fprintf(stderr, "[sfw] pcg: %lld solves, mean %.2f iterations, max %d\n", n_it, (double)sum_it / n_it, max_it);
        o->stats[6] = B;
        o->stats[7] = std::chrono::duration<double>(clk::now() - t_begin).count();
    }
    if (ce != cudaSuccess) return fail(SFW_ECUDA, std::string("ROM build: ") + cudaGetErrorString(ce), errbuf, errlen);
    if (rc) {
        std::string msg = "offline stage failed for " + std::to_string(errors.size()) + " subdomain(s):";
        for (auto& e : errors) msg += "\n  " + e;
        return fail(rc, msg, errbuf, errlen);
    }
    return 0;
}
