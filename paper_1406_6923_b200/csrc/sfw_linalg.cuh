// Small dense linear algebra building blocks for the ROM build (sm_100a):
//   * batched fp64 GEMM on the DMMA tensor pipe (mma.sync.m8n8k4.f64)
//   * CTA-cooperative w x w kernels in shared memory: Cholesky, triangular
//     inverse, LU with partial pivoting (LAPACK gesv semantics), one-sided
//     Jacobi SVD (2-norm condition numbers as numpy.linalg.cond computes them).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sfw {

// ---------------------------------------------------------------------------
// batched DGEMM: C[b] = alpha * op(A[b]) * B[b] + beta * C[b], column-major.
//   op(A) = A (M x K, lda)        when TA = false
//   op(A) = A^T (A is K x M, lda) when TA = true
struct GemmArgs {
    int M, N, K;
    double alpha, beta;
    const double* A;
    long long lda, sA;
    const double* B;
    long long ldb, sB;
    double* C;
    long long ldc, sC;
};

__device__ __forceinline__ void dmma8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

#ifndef SFW_DGEMM_PAD
#define SFW_DGEMM_PAD 4
#endif
template <bool TA>
__global__ void __launch_bounds__(128) k_dgemm(const GemmArgs g) {
    constexpr int BM = 64, BN = 64, BK = 16, PAD = SFW_DGEMM_PAD;  // row stride = 4 mod 16 doubles: conflict-free fragments
    __shared__ __align__(16) double As[2][BK][BM + PAD];
    __shared__ __align__(16) double Bs[2][BK][BN + PAD];
    const int b = blockIdx.z;
    const double* A = g.A + (size_t)b * g.sA;
    const double* B = g.B + (size_t)b * g.sB;
    double* C = g.C + (size_t)b * g.sC;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double ra[8], rb[8];
    auto gload = [&](int k0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int idx = tid + e * 128;
            int m, k;
            if (!TA) {
                m = idx % BM;
                k = idx / BM;
            } else {
                k = idx % BK;
                m = idx / BK;
            }
            const int gm = m0 + m, gk = k0 + k;
            ra[e] = (gm < g.M && gk < g.K) ? (TA ? A[gk + (size_t)gm * g.lda] : A[gm + (size_t)gk * g.lda]) : 0.0;
            const int kb = idx % BK, nb = idx / BK;
            const int gn = n0 + nb, gkb = k0 + kb;
            rb[e] = (gn < g.N && gkb < g.K) ? B[gkb + (size_t)gn * g.ldb] : 0.0;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int idx = tid + e * 128;
            if (!TA)
                As[buf][idx / BM][idx % BM] = ra[e];
            else
                As[buf][idx % BK][idx / BK] = ra[e];
            Bs[buf][idx % BK][idx / BK] = rb[e];
        }
    };
    const int nk = (g.K + BK - 1) / BK;
    gload(0);
    sstore(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) gload((kt + 1) * BK);
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[buf][kk + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][kk + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j], af[i], bf[j]);
        }
        if (kt + 1 < nk) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int gm = m0 + wm + i * 8 + (lane >> 2);
                const int gn = n0 + wn + j * 8 + (lane & 3) * 2 + h;
                if (gm < g.M && gn < g.N) {
                    double* cp = C + gm + (size_t)gn * g.ldc;
                    const double v = g.alpha * acc[i][j][h];
                    *cp = (g.beta != 0.0) ? v + g.beta * *cp : v;
                }
            }
}

// ---------------------------------------------------------------------------
// k_dgemm2: the same batched C = alpha op(A) B + beta C, with the tiles moved global -> shared by
// cp.async (16-byte chunks, zero-filled at the edges) through a 3-stage ring, so no register
// staging and two k-tiles in flight while the DMMA loop runs.  Shared layouts are chosen for
// conflict-free fragment reads: A as [k][m] (row stride 68) when A is column-major in m, else
// [m][k] (row stride 20); B as [n][k] (row stride 20).  Needs 16-byte aligned operands with even
// leading dimensions (the host wrapper checks and otherwise uses k_dgemm).
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int DG2_BM = 64, DG2_BN = 64, DG2_BK = 16, DG2_NS = 3, DG2_LDM = 68, DG2_LDK = 20;
constexpr int DG2_ASZ = DG2_BK * DG2_LDM > DG2_BM * DG2_LDK ? DG2_BK * DG2_LDM : DG2_BM * DG2_LDK;
constexpr int DG2_BSZ = DG2_BN * DG2_LDK;
constexpr size_t DG2_SMEM = (size_t)DG2_NS * (DG2_ASZ + DG2_BSZ) * 8;

template <bool TA>
__global__ void __launch_bounds__(128) k_dgemm2(const GemmArgs g) {
    extern __shared__ __align__(16) double dsm[];
    double* As = dsm;                         // [NS][ASZ]
    double* Bs = dsm + DG2_NS * DG2_ASZ;      // [NS][BSZ]
    const int b = blockIdx.z;
    const double* A = g.A + (size_t)b * g.sA;
    const double* B = g.B + (size_t)b * g.sB;
    double* C = g.C + (size_t)b * g.sC;
    const int m0 = blockIdx.y * DG2_BM, n0 = blockIdx.x * DG2_BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int nk = (g.K + DG2_BK - 1) / DG2_BK;
    auto issue = [&](int kt, int buf) {
        const int k0 = kt * DG2_BK;
        double* as = As + buf * DG2_ASZ;
        double* bs = Bs + buf * DG2_BSZ;
#pragma unroll
        for (int e = 0; e < 4; ++e) {  // 512 chunks of A, 4 per thread
            const int c = tid + e * 128;
            if (!TA) {  // A column-major (m fastest): chunk = 2 m at one k
                const int k = c >> 5, m = (c & 31) * 2;
                const int gm = m0 + m, gk = k0 + k;
                const int valid = (gk < g.K) ? max(0, min(2, g.M - gm)) : 0;
                cp_async16(as + k * DG2_LDM + m, valid ? A + gm + (size_t)gk * g.lda : A, 8 * valid);
            } else {    // A^T: k fastest: chunk = 2 k at one m
                const int m = c >> 3, k = (c & 7) * 2;
                const int gm = m0 + m, gk = k0 + k;
                const int valid = (gm < g.M) ? max(0, min(2, g.K - gk)) : 0;
                cp_async16(as + m * DG2_LDK + k, valid ? A + gk + (size_t)gm * g.lda : A, 8 * valid);
            }
            {  // B (k fastest): chunk = 2 k at one n
                const int n = c >> 3, k = (c & 7) * 2;
                const int gn = n0 + n, gk = k0 + k;
                const int valid = (gn < g.N) ? max(0, min(2, g.K - gk)) : 0;
                cp_async16(bs + n * DG2_LDK + k, valid ? B + gk + (size_t)gn * g.ldb : B, 8 * valid);
            }
        }
    };
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int s = 0; s < DG2_NS - 1; ++s) {
        if (s < nk) issue(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<DG2_NS - 2>();
        __syncthreads();  // stage kt landed for every thread; everyone finished computing kt-1
        if (kt + DG2_NS - 1 < nk) issue(kt + DG2_NS - 1, (kt + DG2_NS - 1) % DG2_NS);
        cp_async_commit();
        const double* as = As + (kt % DG2_NS) * DG2_ASZ;
        const double* bs = Bs + (kt % DG2_NS) * DG2_BSZ;
#pragma unroll
        for (int kk = 0; kk < DG2_BK; kk += 4) {
            double af[4], bf[4];
            const int k = kk + (lane & 3);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int m = wm + i * 8 + (lane >> 2);
                af[i] = TA ? as[m * DG2_LDK + k] : as[k * DG2_LDM + m];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = bs[(wn + j * 8 + (lane >> 2)) * DG2_LDK + k];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma8x8x4(acc[i][j], af[i], bf[j]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int gm = m0 + wm + i * 8 + (lane >> 2);
                const int gn = n0 + wn + j * 8 + (lane & 3) * 2 + h;
                if (gm < g.M && gn < g.N) {
                    double* cp = C + gm + (size_t)gn * g.ldc;
                    const double v = g.alpha * acc[i][j][h];
                    *cp = (g.beta != 0.0) ? v + g.beta * *cp : v;
                }
            }
}

// ---------------------------------------------------------------------------
// CTA-cooperative dense helpers on w x w row-major matrices in shared memory.
// All routines must be called by every thread of the CTA.

__device__ __forceinline__ double block_sum(double v, double* red) {
    // fixed-order block reduction (warp butterfly, then warps in order by thread 0)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = red[0];
        for (int i = 1; i < nw; ++i) t += red[i];
        red[32] = t;
    }
    __syncthreads();
    return red[32];
}

__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = red[0];
        for (int i = 1; i < nw; ++i) t = fmax(t, red[i]);
        red[32] = t;
    }
    __syncthreads();
    return red[32];
}

// C = op(A) op(B), all n x n row-major in smem; C must not alias A or B.
__device__ inline void sm_matmul(const double* A, bool ta, const double* B, bool tb, double* C, int n) {
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        const int i = idx / n, j = idx % n;
        double s = 0.0;
        for (int k = 0; k < n; ++k) {
            const double a = ta ? A[k * n + i] : A[i * n + k];
            const double b = tb ? B[j * n + k] : B[k * n + j];
            s = fma(a, b, s);
        }
        C[idx] = s;
    }
    __syncthreads();
}

// In-place LU with partial pivoting (getrf); returns false if exactly singular.
__device__ inline bool sm_lu(double* A, int* piv, int n, int* flag) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int c = 0; c < n; ++c) {
        if (threadIdx.x == 0) {
            int pr = c;
            double best = fabs(A[c * n + c]);
            for (int r = c + 1; r < n; ++r) {
                const double v = fabs(A[r * n + c]);
                if (v > best) {
                    best = v;
                    pr = r;
                }
            }
            piv[c] = pr;
            if (best == 0.0) *flag = 1;
        }
        __syncthreads();
        const int pr = piv[c];
        if (pr != c)
            for (int k = threadIdx.x; k < n; k += blockDim.x) {
                const double t = A[c * n + k];
                A[c * n + k] = A[pr * n + k];
                A[pr * n + k] = t;
            }
        __syncthreads();
        const double d = A[c * n + c];
        for (int r = c + 1 + threadIdx.x; r < n; r += blockDim.x) A[r * n + c] = (d != 0.0) ? A[r * n + c] / d : 0.0;
        __syncthreads();
        const int rem = n - c - 1;
        for (int idx = threadIdx.x; idx < rem * rem; idx += blockDim.x) {
            const int r = c + 1 + idx / rem, k = c + 1 + idx % rem;
            A[r * n + k] = fma(-A[r * n + c], A[c * n + k], A[r * n + k]);
        }
        __syncthreads();
    }
    const bool ok = (*flag == 0);
    __syncthreads();
    return ok;
}

// Solve (LU) X = B in place, B is n x nrhs row-major (getrs).
__device__ inline void sm_lu_solve(const double* LU, const int* piv, double* B, int n, int nrhs) {
    for (int j = threadIdx.x; j < nrhs; j += blockDim.x) {
        for (int c = 0; c < n; ++c) {
            const int pr = piv[c];
            if (pr != c) {
                const double t = B[c * nrhs + j];
                B[c * nrhs + j] = B[pr * nrhs + j];
                B[pr * nrhs + j] = t;
            }
        }
        for (int r = 0; r < n; ++r) {
            double s = B[r * nrhs + j];
            for (int k = 0; k < r; ++k) s = fma(-LU[r * n + k], B[k * nrhs + j], s);
            B[r * nrhs + j] = s;
        }
        for (int r = n - 1; r >= 0; --r) {
            double s = B[r * nrhs + j];
            for (int k = r + 1; k < n; ++k) s = fma(-LU[r * n + k], B[k * nrhs + j], s);
            B[r * nrhs + j] = s / LU[r * n + r];
        }
    }
    __syncthreads();
}

// 2-norm condition number sigma_max / sigma_min of the n x n matrix A (left
// untouched) by one-sided Jacobi SVD on a copy W (n x n workspace).  Columns
// are orthogonalised pairwise in a fixed round-robin order; returns +inf for a
// (numerically) singular matrix.
__device__ inline double sm_cond2(const double* A, double* W, int n, double* red, int* flag) {
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) W[i] = A[i];
    __syncthreads();
    const int m = (n % 2) ? n + 1 : n;  // tournament size (dummy player if n is odd)
    const int rounds = m - 1;
    for (int sweep = 0; sweep < 40; ++sweep) {
        if (threadIdx.x == 0) *flag = 0;
        __syncthreads();
        for (int rd = 0; rd < rounds; ++rd) {
            // round-robin tournament pairing (fixed order)
            for (int pi = threadIdx.x >> 5; pi < (m / 2); pi += (blockDim.x >> 5)) {
                // circle-method round robin: every pair exactly once per sweep, disjoint within a round
                int a, b;
                if (pi == 0) {
                    a = m - 1;
                    b = rd;
                } else {
                    a = (rd + pi) % (m - 1);
                    b = (rd - pi + m - 1) % (m - 1);
                }
                if (a >= n || b >= n || a == b) continue;
                if (a > b) {
                    const int t = a;
                    a = b;
                    b = t;
                }
                const int lane = threadIdx.x & 31;
                double al = 0, be = 0, ga = 0;
                for (int r = lane; r < n; r += 32) {
                    const double x = W[r * n + a], y = W[r * n + b];
                    al = fma(x, x, al);
                    be = fma(y, y, be);
                    ga = fma(x, y, ga);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (fabs(ga) > 1e-15 * sqrt(al * be) && ga != 0.0) {
                    const double zeta = (be - al) / (2.0 * ga);
                    const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
                    for (int r = lane; r < n; r += 32) {
                        const double x = W[r * n + a], y = W[r * n + b];
                        W[r * n + a] = cs * x - sn * y;
                        W[r * n + b] = sn * x + cs * y;
                    }
                    if (lane == 0) *flag = 1;
                }
            }
            __syncthreads();
        }
        if (*flag == 0) break;
        __syncthreads();
    }
    __syncthreads();
    double smax = 0.0, smin = 1e308;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < n; ++r) s = fma(W[r * n + j], W[r * n + j], s);
        s = sqrt(s);
        smax = fmax(smax, s);
        smin = fmin(smin, s);
    }
    smax = block_max(smax, red);
    smin = -block_max(-smin, red);
    if (!(smin > 0.0)) return __longlong_as_double(0x7ff0000000000000LL);
    return smax / smin;
}

// Condition check for "cond2(A) > limit" (numpy.linalg.cond semantics) from an existing
// LU factorisation of A (or A^T): cond_F = |A|_F |A^-1|_F satisfies cond_F/n <= cond2 <= cond_F,
// so the decision is exact unless cond_F falls in [limit, n*limit], where the exact one-sided
// Jacobi SVD of A decides.  Returns a value on the same side of limit as cond2(A).
// Wk, Wk2: n x n workspaces; A is left untouched.
__device__ inline double sm_cond2_check(const double* A, const double* LU, const int* piv, double* Wk, double* Wk2,
                                        int n, double limit, double* red, int* flag) {
    double fa = 0.0;
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
        fa = fma(A[i], A[i], fa);
        Wk[i] = (i / n == i % n) ? 1.0 : 0.0;
    }
    fa = block_sum(fa, red);
    sm_lu_solve(LU, piv, Wk, n, n);  // Wk = A^-1 (or A^-T): same Frobenius norm
    double fi = 0.0;
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) fi = fma(Wk[i], Wk[i], fi);
    fi = block_sum(fi, red);
    const double cf = sqrt(fa) * sqrt(fi);
    if (!(cf == cf) || isinf(cf)) return __longlong_as_double(0x7ff0000000000000LL);
    if (cf <= limit) return cf;
    if (cf / n > limit) return cf / n;
    return sm_cond2(A, Wk2, n, red, flag);
}

}  // namespace sfw
