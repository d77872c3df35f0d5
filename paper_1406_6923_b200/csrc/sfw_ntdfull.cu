// Transfer maps of an operator given explicitly (reference ntd.py:62-115,
// 188-202): ntd_full (the sparse N x N subdomain operator) and ntd_reduced (the dense projected
// pair), both  M(w) = sym(F^T (A + w^2 I)^-1 F).
//
// One CTA per frequency.  The shifted matrix is scattered from CSR into LAPACK band storage
// (kl = ku = the sparsity half-bandwidth: P^2 = 289 for the 17^3 subdomain in natural order,
// n-1 for a dense pair) and factored by band LU with partial pivoting in LAPACK dgbtf2 order
// (first maximal |pivot|, reciprocal scaling, fill tracked by ju), then solved for the w
// right-hand sides in dgbtrs order.  The reference factors with SuperLU (COLAMD ordering,
// threshold pivoting), so the two agree to the conditioning of A + w^2 I, not bit for bit.
// The relative residual ||A X + w^2 X - F||_F / ||F||_F is computed on the device from the CSR
// operator; the host applies the reference's resonance test (RESONANCE_RTOL) to it.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "sfw_common.cuh"

namespace sfw {

struct GbArgs {
    int n, kl, ku, ldab, w;
    const int* rp;
    const int* ci;
    const double* val;
    const double* F;       // [n][w] row-major
    const double* omega;   // [n_sys]
    double* ab;            // [n_sys][n][ldab]: column j at ab + j * ldab, entry (i, j) at kl + ku + i - j
    int* piv;              // [n_sys][n]
    double* X;             // [n_sys][n][w]
    double* out;           // [n_sys][w][w]
    double* resid;         // [n_sys]
    int* status;           // [n_sys]: 0 ok, j+1 zero pivot in column j
};

__device__ inline double gb_block_sum(double v, double* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];  // fixed order
        red[32] = t;
    }
    __syncthreads();
    return red[32];
}

__global__ void __launch_bounds__(1024) k_gb_ntd(GbArgs a) {
    const int sys = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const int n = a.n, kl = a.kl, ku = a.ku, ldab = a.ldab, w = a.w, kv = kl + ku;
    double* ab = a.ab + (size_t)sys * n * ldab;
    int* piv = a.piv + (size_t)sys * n;
    double* X = a.X + (size_t)sys * n * w;
    const double om = a.omega[sys];
    const double wsq = om * om;
    __shared__ double red[33];
    __shared__ int s_jp, s_bad;
    __shared__ double s_pv;
    // ---- A + w^2 I into band storage; X = F -----------------------------------------
    for (size_t i = tid; i < (size_t)n * ldab; i += nt) ab[i] = 0.0;
    for (size_t i = tid; i < (size_t)n * w; i += nt) X[i] = a.F[i];
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int i = tid; i < n; i += nt)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int j = a.ci[k];
            ab[(size_t)j * ldab + kv + i - j] = a.val[k];
        }
    __syncthreads();
    for (int i = tid; i < n; i += nt) ab[(size_t)i * ldab + kv] += wsq;  // matrix + wsq * identity
    __syncthreads();
    // ---- dgbtf2 ----------------------------------------------------------------------
    int ju = 0;
    for (int j = 0; j < n; ++j) {
        const int km = min(kl, n - 1 - j);
        double* cj = ab + (size_t)j * ldab + kv;  // cj[r] = entry (j + r, j)
        if (tid < 32) {  // first index of max |a| over rows j .. j + km (idamax)
            double best = -1.0;
            int bi = 0;
            for (int r = tid; r <= km; r += 32) {
                const double v = fabs(cj[r]);
                if (v > best) {
                    best = v;
                    bi = r;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (tid == 0) {
                s_jp = bi;
                s_pv = cj[bi];
            }
        }
        __syncthreads();
        const int jp = s_jp;
        if (tid == 0) piv[j] = j + jp;
        if (s_pv == 0.0) {  // exactly singular column: LAPACK records info and goes on
            if (tid == 0 && s_bad == 0) s_bad = j + 1;
            __syncthreads();
            continue;
        }
        ju = max(ju, min(j + ku + jp, n - 1));
        if (jp != 0)  // interchange rows j and j + jp over columns j .. ju
            for (int c = j + tid; c <= ju; c += nt) {
                double* col = ab + (size_t)c * ldab + kv - c;
                const double t = col[j + jp];
                col[j + jp] = col[j];
                col[j] = t;
            }
        __syncthreads();
        if (km > 0) {
            const double rp = 1.0 / cj[0];
            for (int r = 1 + tid; r <= km; r += nt) cj[r] *= rp;
            __syncthreads();
            const int ncol = ju - j;  // rank-1 update of rows j+1 .. j+km, columns j+1 .. ju
            const long long tot = (long long)ncol * km;
            for (long long q = tid; q < tot; q += nt) {
                const int c = j + 1 + (int)(q / km), r = 1 + (int)(q % km);
                double* col = ab + (size_t)c * ldab + kv - c;
                col[j + r] -= cj[r] * col[j];
            }
        }
        __syncthreads();
    }
    // ---- dgbtrs (no transpose): L then U ----------------------------------------------
    for (int j = 0; j < n - 1; ++j) {
        const int lm = min(kl, n - 1 - j), l = piv[j];
        if (l != j)
            for (int c = tid; c < w; c += nt) {
                const double t = X[(size_t)l * w + c];
                X[(size_t)l * w + c] = X[(size_t)j * w + c];
                X[(size_t)j * w + c] = t;
            }
        __syncthreads();
        const double* cj = ab + (size_t)j * ldab + kv;
        for (int q = tid; q < lm * w; q += nt) {
            const int r = 1 + q / w, c = q % w;
            X[(size_t)(j + r) * w + c] -= cj[r] * X[(size_t)j * w + c];
        }
        __syncthreads();
    }
    for (int j = n - 1; j >= 0; --j) {
        const double* col = ab + (size_t)j * ldab + kv - j;  // col[i] = entry (i, j)
        for (int c = tid; c < w; c += nt) X[(size_t)j * w + c] /= col[j];
        __syncthreads();
        const int i0 = max(0, j - kv);
        for (int q = tid; q < (j - i0) * w; q += nt) {
            const int i = i0 + q / w, c = q % w;
            X[(size_t)i * w + c] -= col[i] * X[(size_t)j * w + c];
        }
        __syncthreads();
    }
    // ---- residual (ntd.py:77-78) and sym(F^T X) -----------------------------------------
    double rr = 0.0, ff = 0.0;
    for (size_t q = tid; q < (size_t)n * w; q += nt) {
        const int i = (int)(q / w), c = (int)(q % w);
        double s = 0.0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) s += a.val[k] * X[(size_t)a.ci[k] * w + c];
        const double r = s + wsq * X[q] - a.F[q];
        rr = fma(r, r, rr);
        ff = fma(a.F[q], a.F[q], ff);
    }
    rr = gb_block_sum(rr, red);
    ff = gb_block_sum(ff, red);
    double* o = a.out + (size_t)sys * w * w;
    for (int q = tid; q < w * w; q += nt) {
        const int r = q / w, c = q % w;
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = fma(a.F[(size_t)i * w + r], X[(size_t)i * w + c], s);
        o[q] = s;
    }
    __syncthreads();
    for (int q = tid; q < w * w; q += nt) {
        const int r = q / w, c = q % w;
        if (r < c) {
            const double s = 0.5 * (o[q] + o[(size_t)c * w + r]);
            o[q] = s;
            o[(size_t)c * w + r] = s;
        }
    }
    if (tid == 0) {
        a.resid[sys] = sqrt(rr) / fmax(sqrt(ff), 1e-300);
        a.status[sys] = s_bad;
    }
}

}  // namespace sfw

using namespace sfw;

extern "C" int sfw_ntd_operator(int n, const int* row_ptr, const int* col_idx, const double* vals, int w,
                                const double* F, int n_omega, const double* omegas, double* out, double* resid,
                                int* status, char* errbuf, int errlen) {
    if (n < 1 || w < 1 || n_omega < 0) return fail(SFW_ECONFIG, "bad transfer-map problem shape", errbuf, errlen);
    if (n_omega == 0) return 0;
    const int nnz = row_ptr[n];
    int kl = 0;
    for (int i = 0; i < n; ++i)
        for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            const int j = col_idx[k];
            if (j < 0 || j >= n) return fail(SFW_ECONFIG, "column index out of range", errbuf, errlen);
            kl = std::max(kl, std::abs(i - j));
        }
    const int ku = kl, ldab = 2 * kl + ku + 1;
    const size_t per = (size_t)n * ldab * 8 + (size_t)n * w * 8 + (size_t)n * 4;
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const int batch = (int)std::max<size_t>(1, std::min<size_t>((size_t)n_omega, (free_b / 2) / per));
    int *drp = nullptr, *dci = nullptr, *dpiv = nullptr, *dst = nullptr;
    double *dval = nullptr, *dF = nullptr, *dom = nullptr, *dab = nullptr, *dX = nullptr, *dout = nullptr,
           *dres = nullptr;
    auto cleanup = [&]() {
        cudaFree(drp);
        cudaFree(dci);
        cudaFree(dpiv);
        cudaFree(dst);
        cudaFree(dval);
        cudaFree(dF);
        cudaFree(dom);
        cudaFree(dab);
        cudaFree(dX);
        cudaFree(dout);
        cudaFree(dres);
    };
#define GB_TRY(x)                                                   \
    do {                                                            \
        cudaError_t e_ = (x);                                       \
        if (e_ != cudaSuccess) {                                    \
            cleanup();                                              \
            return fail(SFW_ECUDA, cudaGetErrorString(e_), errbuf, errlen); \
        }                                                           \
    } while (0)
    GB_TRY(cudaMalloc(&drp, (n + 1) * 4));
    GB_TRY(cudaMalloc(&dci, std::max(nnz, 1) * 4));
    GB_TRY(cudaMalloc(&dval, std::max(nnz, 1) * 8));
    GB_TRY(cudaMalloc(&dF, (size_t)n * w * 8));
    GB_TRY(cudaMalloc(&dom, n_omega * 8));
    GB_TRY(cudaMalloc(&dab, (size_t)batch * n * ldab * 8));
    GB_TRY(cudaMalloc(&dX, (size_t)batch * n * w * 8));
    GB_TRY(cudaMalloc(&dpiv, (size_t)batch * n * 4));
    GB_TRY(cudaMalloc(&dout, (size_t)n_omega * w * w * 8));
    GB_TRY(cudaMalloc(&dres, n_omega * 8));
    GB_TRY(cudaMalloc(&dst, n_omega * 4));
    GB_TRY(sfw_h2d(drp, row_ptr, (n + 1) * 4));
    if (nnz) {
        GB_TRY(sfw_h2d(dci, col_idx, nnz * 4));
        GB_TRY(sfw_h2d(dval, vals, (size_t)nnz * 8));
    }
    GB_TRY(sfw_h2d(dF, F, (size_t)n * w * 8));
    GB_TRY(sfw_h2d(dom, omegas, n_omega * 8));
    for (int s0 = 0; s0 < n_omega; s0 += batch) {
        const int nb = std::min(batch, n_omega - s0);
        GbArgs ga{n, kl, ku, ldab, w, drp, dci, dval, dF, dom + s0, dab, dpiv, dX,
                  dout + (size_t)s0 * w * w, dres + s0, dst + s0};
        k_gb_ntd<<<nb, 1024>>>(ga);
        GB_TRY(cudaGetLastError());
    }
    GB_TRY(cudaDeviceSynchronize());
    GB_TRY(cudaMemcpy(out, dout, (size_t)n_omega * w * w * 8, cudaMemcpyDeviceToHost));
    GB_TRY(cudaMemcpy(resid, dres, n_omega * 8, cudaMemcpyDeviceToHost));
    GB_TRY(cudaMemcpy(status, dst, n_omega * 4, cudaMemcpyDeviceToHost));
#undef GB_TRY
    cleanup();
    return 0;
}
