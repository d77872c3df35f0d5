// Transfer maps of an operator given explicitly (reference ntd.py:62-115,
// 188-202): ntd_full (the sparse N x N subdomain operator) and ntd_reduced (the dense projected
// pair), both  M(w) = sym(F^T (A + w^2 I)^-1 F).
//
// A gang of CTAs per frequency (one CTA when there are at least as many frequencies as SMs; see k_gb_ntd).
// The shifted matrix is scattered from CSR into LAPACK band storage
// (kl = ku = the sparsity half-bandwidth: P^2 = 289 for the 17^3 subdomain in natural order,
// n-1 for a dense pair) and factored by band LU with partial pivoting in LAPACK dgbtf2 order
// (first maximal |pivot|, reciprocal scaling, fill tracked by ju), then solved for the w
// right-hand sides in dgbtrs order.  The reference factors with SuperLU (COLAMD ordering,
// threshold pivoting), so the two agree to the conditioning of A + w^2 I, not bit for bit.
// The relative residual ||A X + w^2 X - F||_F / ||F||_F is computed on the device from the CSR
// operator; the host applies the reference's resonance test (RESONANCE_RTOL) to it.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
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
    int G;                 // CTAs per system (gang)
    unsigned int* ctr;     // [n_sys] gang barrier counters (zeroed)
    double* part;          // [n_sys][G][2] residual partials
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

// A gang of G CTAs factors and solves one system (G = 1 when there are at least as many frequencies
// as SMs).  Column c of the band belongs to CTA c mod G, which alone interchanges and updates it; every
// CTA reads the pivot column (through L2), finds the pivot and forms the scaled multipliers in its own
// shared memory, so one gang barrier per column is enough.  The solves split the w right-hand sides over
// the gang and need no barrier at all.  Entries written by another CTA are read with ld.global.cg.
__global__ void __launch_bounds__(1024) k_gb_ntd(GbArgs a) {
    extern __shared__ double sl[];  // [kl + 1] pivot column: entry (j + r, j), then the multipliers
    const int G = a.G;
    const int sys = blockIdx.x / G, g = blockIdx.x % G, tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    const int n = a.n, kl = a.kl, ku = a.ku, ldab = a.ldab, w = a.w, kv = kl + ku;
    double* ab = a.ab + (size_t)sys * n * ldab;
    int* piv = a.piv + (size_t)sys * n;
    double* X = a.X + (size_t)sys * n * w;
    const double om = a.omega[sys];
    const double wsq = om * om;
    __shared__ double red[33];
    __shared__ int s_jp, s_bad;
    __shared__ double s_pv;
    unsigned int* ctr = a.ctr + sys;
    unsigned int bar = 0;
    auto gang_sync = [&]() {
        __syncthreads();
        if (G > 1) {
            bar += (unsigned int)G;
            if (tid == 0) {
                grid_arrive(ctr);
                grid_wait(ctr, bar);
            }
            __syncthreads();
        }
    };
    const int mw = (w - g + G - 1) / G;  // this CTA's right-hand sides: c = g, g + G, ...
    // ---- A + w^2 I into band storage; X = F (own right-hand sides) ------------------------
    for (size_t i = (size_t)g * nt + tid; i < (size_t)n * ldab; i += (size_t)G * nt) ab[i] = 0.0;
    for (size_t q = tid; q < (size_t)n * mw; q += nt) {
        const size_t i = q / mw;
        const int c = g + (int)(q % mw) * G;
        X[i * w + c] = a.F[i * w + c];
    }
    if (tid == 0) s_bad = 0;
    gang_sync();
    for (int i = g * nt + tid; i < n; i += G * nt)
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) {
            const int j = a.ci[k];
            ab[(size_t)j * ldab + kv + i - j] = a.val[k];
        }
    gang_sync();
    for (int i = g * nt + tid; i < n; i += G * nt) {  // matrix + wsq * identity
        double* d = ab + (size_t)i * ldab + kv;
        *d = __ldcg(d) + wsq;
    }
    gang_sync();
    // ---- dgbtf2 ----------------------------------------------------------------------
    int ju = 0;
    for (int j = 0; j < n; ++j) {
        const int km = min(kl, n - 1 - j);
        double* cj = ab + (size_t)j * ldab + kv;  // cj[r] = entry (j + r, j)
        for (int r = tid; r <= km; r += nt) sl[r] = __ldcg(cj + r);
        __syncthreads();
        if (tid < 32) {  // first index of max |a| over rows j .. j + km (idamax)
            double best = -1.0;
            int bi = 0;
            for (int r = tid; r <= km; r += 32) {
                const double v = fabs(sl[r]);
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
                s_pv = sl[bi];
            }
        }
        __syncthreads();
        const int jp = s_jp;
        if (g == 0 && tid == 0) piv[j] = j + jp;
        if (s_pv == 0.0) {  // exactly singular column: LAPACK records info and goes on (every CTA alike)
            if (tid == 0 && s_bad == 0) s_bad = j + 1;
            __syncthreads();
            continue;
        }
        ju = max(ju, min(j + ku + jp, n - 1));
        if (tid == 0 && jp != 0) {  // rows j and j + jp of the pivot column
            const double t = sl[jp];
            sl[jp] = sl[0];
            sl[0] = t;
        }
        __syncthreads();
        if (km > 0) {
            const double rp = 1.0 / sl[0];
            __syncthreads();
            for (int r = 1 + tid; r <= km; r += nt) sl[r] *= rp;
            __syncthreads();
        }
        // own columns j+1 .. ju: interchange rows j and j + jp, then the rank-1 update of rows j+1 .. j+km
        // (one warp per column, lanes along the contiguous rows)
        const int c0 = j + 1 + ((g - (j + 1) % G) % G + G) % G;
        for (int c = c0 + warp * G; c <= ju; c += nw * G) {
            double* col = ab + (size_t)c * ldab + kv - c;
            double top = 0.0, low = 0.0;  // entries (j, c) and (j + jp, c) after the interchange
            if (lane == 0) {
                top = __ldcg(col + j);
                if (jp != 0) {
                    low = top;
                    top = __ldcg(col + j + jp);
                    col[j + jp] = low;
                    col[j] = top;
                }
            }
            top = __shfl_sync(0xffffffffu, top, 0);
            low = __shfl_sync(0xffffffffu, low, 0);
            for (int r = 1 + lane; r <= km; r += 32) {
                const double v = (jp != 0 && r == jp) ? low : __ldcg(col + j + r);
                col[j + r] = v - sl[r] * top;
            }
        }
        if (km > 0) {
            gang_sync();  // every CTA has read column j: its owner may now store it (pivot on top, multipliers below)
            if (j % G == g)
                for (int r = tid; r <= km; r += nt) cj[r] = sl[r];
            __syncthreads();
        }
    }
    gang_sync();
    // ---- dgbtrs (no transpose): L then U, own right-hand sides ---------------------------
    for (int j = 0; j < n - 1; ++j) {
        const int lm = min(kl, n - 1 - j), l = __ldcg(piv + j);
        if (l != j)
            for (int ci = tid; ci < mw; ci += nt) {
                const int c = g + ci * G;
                const double t = X[(size_t)l * w + c];
                X[(size_t)l * w + c] = X[(size_t)j * w + c];
                X[(size_t)j * w + c] = t;
            }
        __syncthreads();
        const double* cj = ab + (size_t)j * ldab + kv;
        for (int q = tid; q < lm * mw; q += nt) {
            const int r = 1 + q / mw, c = g + (q % mw) * G;
            X[(size_t)(j + r) * w + c] -= __ldcg(cj + r) * X[(size_t)j * w + c];
        }
        __syncthreads();
    }
    for (int j = n - 1; j >= 0; --j) {
        const double* col = ab + (size_t)j * ldab + kv - j;  // col[i] = entry (i, j)
        const double pj = __ldcg(col + j);
        for (int ci = tid; ci < mw; ci += nt) X[(size_t)j * w + g + ci * G] /= pj;
        __syncthreads();
        const int i0 = max(0, j - kv);
        for (int q = tid; q < (j - i0) * mw; q += nt) {
            const int i = i0 + q / mw, c = g + (q % mw) * G;
            X[(size_t)i * w + c] -= __ldcg(col + i) * X[(size_t)j * w + c];
        }
        __syncthreads();
    }
    // ---- residual (ntd.py:77-78) and sym(F^T X) -----------------------------------------
    double rr = 0.0, ff = 0.0;
    for (size_t q = tid; q < (size_t)n * mw; q += nt) {
        const int i = (int)(q / mw), c = g + (int)(q % mw) * G;
        double s = 0.0;
        for (int k = a.rp[i]; k < a.rp[i + 1]; ++k) s += a.val[k] * X[(size_t)a.ci[k] * w + c];
        const double f = a.F[(size_t)i * w + c];
        const double r = s + wsq * X[(size_t)i * w + c] - f;
        rr = fma(r, r, rr);
        ff = fma(f, f, ff);
    }
    rr = gb_block_sum(rr, red);
    ff = gb_block_sum(ff, red);
    if (tid == 0) {
        a.part[((size_t)sys * G + g) * 2] = rr;
        a.part[((size_t)sys * G + g) * 2 + 1] = ff;
    }
    double* o = a.out + (size_t)sys * w * w;
    for (int q = tid; q < w * mw; q += nt) {
        const int r = q / mw, c = g + (q % mw) * G;
        double s = 0.0;
        for (int i = 0; i < n; ++i) s = fma(a.F[(size_t)i * w + r], X[(size_t)i * w + c], s);
        o[(size_t)r * w + c] = s;
    }
    gang_sync();
    if (g != 0) return;
    for (int q = tid; q < w * w; q += nt) {
        const int r = q / w, c = q % w;
        if (r < c) {
            const double s = 0.5 * (__ldcg(o + q) + __ldcg(o + (size_t)c * w + r));
            o[q] = s;
            o[(size_t)c * w + r] = s;
        }
    }
    if (tid == 0) {
        double tr = 0.0, tf = 0.0;
        for (int k = 0; k < G; ++k) {  // fixed order over the gang
            tr += __ldcg(a.part + ((size_t)sys * G + k) * 2);
            tf += __ldcg(a.part + ((size_t)sys * G + k) * 2 + 1);
        }
        a.resid[sys] = sqrt(tr) / fmax(sqrt(tf), 1e-300);
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
    const size_t batch_mem = std::max<size_t>(1, std::min<size_t>((size_t)n_omega, (free_b / 2) / per));
    // gang size: with fewer frequencies than SMs several CTAs share one system (SFW_NTD_GANG: test hook)
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t gb_smem = (size_t)(kl + 2) * 8;
    int per_sm = 0;
    cudaFuncSetAttribute(k_gb_ntd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb_smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gb_ntd, 1024, gb_smem);
    const int maxco = std::max(1, per_sm * nsm);
    int G = std::max(1, std::min(32, maxco / std::max(1, n_omega)));
    if (const char* e = getenv("SFW_NTD_GANG")) G = std::max(1, std::min(maxco, atoi(e)));
    const int batch = (int)std::max<size_t>(1, std::min<size_t>(batch_mem, (size_t)(maxco / G)));
    int *drp = nullptr, *dci = nullptr, *dpiv = nullptr, *dst = nullptr;
    unsigned int* dctr = nullptr;
    double *dval = nullptr, *dF = nullptr, *dom = nullptr, *dab = nullptr, *dX = nullptr, *dout = nullptr,
           *dres = nullptr, *dpart = nullptr;
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
        cudaFree(dctr);
        cudaFree(dpart);
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
    GB_TRY(cudaMalloc(&dctr, n_omega * 4));
    GB_TRY(cudaMalloc(&dpart, (size_t)n_omega * G * 16));
    GB_TRY(cudaMemset(dctr, 0, n_omega * 4));
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
                  dout + (size_t)s0 * w * w, dres + s0, dst + s0, G, dctr + s0, dpart + (size_t)s0 * G * 2};
        void* args[] = {&ga};  // cooperative: the gang's CTAs wait for each other
        GB_TRY(cudaLaunchCooperativeKernel((const void*)k_gb_ntd, dim3(nb * G), dim3(1024), args, gb_smem, 0));
    }
    GB_TRY(cudaDeviceSynchronize());
    GB_TRY(cudaMemcpy(out, dout, (size_t)n_omega * w * w * 8, cudaMemcpyDeviceToHost));
    GB_TRY(cudaMemcpy(resid, dres, n_omega * 8, cudaMemcpyDeviceToHost));
    GB_TRY(cudaMemcpy(status, dst, n_omega * 4, cudaMemcpyDeviceToHost));
#undef GB_TRY
    cleanup();
    return 0;
}
