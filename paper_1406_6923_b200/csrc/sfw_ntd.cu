// Batched frequency-domain transfer maps of the reduced models (reference
// ntd.py:101-185, sim.py:703-768).
//
// For a model and an angular frequency w the Neumann-to-Dirichlet map M(w) = F*(A + w^2 I)^-1 F
// has two reduced representations the reference cross-checks:
//   tridiag (ntd.py:101-146): block-Lanczos blocks (D_j, B_j, E): backward Schur elimination
//       S <- D_j + w^2 I - B_j^T S^-1 B_j, then M = E^T S^-1 E; a Schur complement with
//       cond_2 > 1e13 switches to one pivoted solve of the assembled (L w)^2 system;
//   chain (ntd.py:149-185): the layer system of the S-fraction coefficients (Gamma, Gamma-hat)
//       with the first Gamma-hat as right-hand side; M = first block of the solution.
// Every (model, w) item is one CTA working on w x w blocks in shared memory (LU with partial
// pivoting = LAPACK gesv semantics, exact cond_2 > limit decisions via sm_cond2_check).  The
// chain form is solved by the same backward block elimination (mathematically the assembled
// solve's first block).  Items whose tridiag Schur chain trips the condition test are solved
// by the assembled fallback kernel (dense LU of the (L w)^2 system in a global workspace).
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "sfw_common.cuh"
#include "sfw_linalg.cuh"

namespace sfw {

struct NtdArgs {
    int form, L, w;
    const double* A;    // tridiag: diag blocks [model][L][w][w]; chain: gammas [model][L][w][w]
    const double* B;    // tridiag: off blocks [model][L-1][w][w]; chain: gamma_hats [model][L][w][w]
    const double* E;    // tridiag: entry block [model][w][w]
    const int* model;   // [item]
    const double* omega;
    double* out;        // [item][w][w]
    int* status;        // [item]: 0 ok, 1 needs the assembled fallback, 2 singular
};

// C = A_s B_s (row-major, n x n), fixed-order fma accumulation
__device__ inline void nt_mm(const double* A, const double* B, double* C, int n) {
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        const int i = idx / n, j = idx % n;
        double s = 0.0;
        for (int k = 0; k < n; ++k) s = fma(A[i * n + k], B[k * n + j], s);
        C[idx] = s;
    }
    __syncthreads();
}

__global__ void k_ntd(const NtdArgs a) {
    extern __shared__ double sm[];
    const int w = a.w, ww = w * w, L = a.L;
    double* S = sm;         // Schur complement
    double* X = S + ww;     // solve workspace / right-hand sides
    double* T = X + ww;     // blocks
    double* W1 = T + ww;    // cond workspaces
    double* W2 = W1 + ww;
    double* LU = W2 + ww;
    int* piv = reinterpret_cast<int*>(LU + ww);
    __shared__ double red[32];
    __shared__ int flag;
    const int item = blockIdx.x, md = a.model[item];
    const double wsq = a.omega[item] * a.omega[item];
    if (a.form == 0) {
        const double* D = a.A + (size_t)md * L * ww;
        const double* Bo = a.B + (size_t)md * (L - 1) * ww;
        for (int i = threadIdx.x; i < ww; i += blockDim.x)
            S[i] = D[(size_t)(L - 1) * ww + i] + ((i / w == i % w) ? wsq : 0.0);
        __syncthreads();
        for (int j = L - 2; j >= 0; --j) {
            for (int i = threadIdx.x; i < ww; i += blockDim.x) LU[i] = S[i];
            __syncthreads();
            const bool nonsing = sm_lu(LU, piv, w, &flag);
            const double cnd = nonsing ? sm_cond2_check(S, LU, piv, W1, W2, w, 1e13, red, &flag)
                                       : __longlong_as_double(0x7ff0000000000000LL);
            if (!(cnd <= 1e13)) {
                if (threadIdx.x == 0) a.status[item] = 1;
                return;
            }
            const double* b = Bo + (size_t)j * ww;
            for (int i = threadIdx.x; i < ww; i += blockDim.x) X[i] = b[i];
            __syncthreads();
            sm_lu_solve(LU, piv, X, w, w);   // X = S^-1 B_j
            __syncthreads();
            for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {  // S = (D_j + w^2 I) - B_j^T X
                const int r = idx / w, c = idx % w;
                double s = 0.0;
                for (int k = 0; k < w; ++k) s = fma(b[k * w + r], X[k * w + c], s);
                T[idx] = (D[(size_t)j * ww + idx] + ((r == c) ? wsq : 0.0)) - s;
            }
            __syncthreads();
            for (int i = threadIdx.x; i < ww; i += blockDim.x) S[i] = T[i];
            __syncthreads();
        }
        for (int i = threadIdx.x; i < ww; i += blockDim.x) LU[i] = S[i];
        __syncthreads();
        const bool nonsing = sm_lu(LU, piv, w, &flag);
        const double cnd = nonsing ? sm_cond2_check(S, LU, piv, W1, W2, w, 1e13, red, &flag)
                                   : __longlong_as_double(0x7ff0000000000000LL);
        if (!(cnd <= 1e13)) {
            if (threadIdx.x == 0) a.status[item] = 1;
            return;
        }
        const double* e = a.E + (size_t)md * ww;
        for (int i = threadIdx.x; i < ww; i += blockDim.x) X[i] = e[i];
        __syncthreads();
        sm_lu_solve(LU, piv, X, w, w);
        __syncthreads();
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {  // T = E^T X
            const int r = idx / w, c = idx % w;
            double s = 0.0;
            for (int k = 0; k < w; ++k) s = fma(e[k * w + r], X[k * w + c], s);
            T[idx] = s;
        }
    } else {
        // chain: rows j of the layer system; backward elimination onto block 0
        const double* G = a.A + (size_t)md * L * ww;
        const double* H = a.B + (size_t)md * L * ww;
        auto diag_block = [&](int j, double* out) {  // w^2 I - H_j (G_j + G_{j-1})
            for (int i = threadIdx.x; i < ww; i += blockDim.x)
                W1[i] = G[(size_t)j * ww + i] + (j > 0 ? G[(size_t)(j - 1) * ww + i] : 0.0);
            __syncthreads();
            nt_mm(H + (size_t)j * ww, W1, W2, w);
            for (int i = threadIdx.x; i < ww; i += blockDim.x) out[i] = ((i / w == i % w) ? wsq : 0.0) - W2[i];
            __syncthreads();
        };
        diag_block(L - 1, S);
        for (int j = L - 2; j >= 0; --j) {
            for (int i = threadIdx.x; i < ww; i += blockDim.x) LU[i] = S[i];
            __syncthreads();
            if (!sm_lu(LU, piv, w, &flag)) {
                if (threadIdx.x == 0) a.status[item] = 2;
                return;
            }
            nt_mm(H + (size_t)(j + 1) * ww, G + (size_t)j * ww, X, w);  // lower block (j+1, j) = H_{j+1} G_j
            sm_lu_solve(LU, piv, X, w, w);                               // X = S^-1 lower
            __syncthreads();
            nt_mm(H + (size_t)j * ww, G + (size_t)j * ww, T, w);        // upper block (j, j+1) = H_j G_j
            diag_block(j, S);                                            // S = D_j (W1, W2 scratch) ...
            nt_mm(T, X, W2, w);                                          // W2 = upper S_{j+1}^-1 lower
            for (int i = threadIdx.x; i < ww; i += blockDim.x) S[i] -= W2[i];  // ... - W2
            __syncthreads();
        }
        for (int i = threadIdx.x; i < ww; i += blockDim.x) LU[i] = S[i];
        __syncthreads();
        if (!sm_lu(LU, piv, w, &flag)) {
            if (threadIdx.x == 0) a.status[item] = 2;
            return;
        }
        for (int i = threadIdx.x; i < ww; i += blockDim.x) X[i] = H[i];  // right-hand side: Gamma-hat_0
        __syncthreads();
        sm_lu_solve(LU, piv, X, w, w);
        __syncthreads();
        for (int i = threadIdx.x; i < ww; i += blockDim.x) T[i] = X[i];
    }
    __syncthreads();
    double* o = a.out + (size_t)item * ww;
    for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {  // 0.5 (M + M^T)
        const int r = idx / w, c = idx % w;
        o[idx] = 0.5 * (T[r * w + c] + T[c * w + r]);
    }
    if (threadIdx.x == 0) a.status[item] = 0;
}

// assembled fallback of the tridiag form (ntd.py:129-146): one pivoted solve of the (L w)^2
// system in a global workspace (rare: only items whose Schur chain is ill-conditioned)
__global__ void k_ntd_assembled(const NtdArgs a, const int* items, double* work) {
    const int w = a.w, ww = w * w, L = a.L, n = L * w;
    const int item = items[blockIdx.x], md = a.model[item];
    const double wsq = a.omega[item] * a.omega[item];
    double* F = work + (size_t)blockIdx.x * ((size_t)n * n + (size_t)n * w + n);
    double* R = F + (size_t)n * n;
    int* piv = reinterpret_cast<int*>(R + (size_t)n * w);
    __shared__ int flag;
    const double* D = a.A + (size_t)md * L * ww;
    const double* Bo = a.B + (size_t)md * (L - 1) * ww;
    const double* e = a.E + (size_t)md * ww;
    for (long long idx = threadIdx.x; idx < (long long)n * n; idx += blockDim.x) {
        const int r = (int)(idx / n), c = (int)(idx % n);
        const int I = r / w, J = c / w, rr = r % w, cc = c % w;
        double v = 0.0;
        if (I == J) v = D[(size_t)I * ww + rr * w + cc] + ((rr == cc) ? wsq : 0.0);
        else if (I == J + 1) v = Bo[(size_t)J * ww + rr * w + cc];            // full[next, blk] = B_j
        else if (J == I + 1) v = Bo[(size_t)I * ww + cc * w + rr];            // full[blk, next] = B_j^T
        F[idx] = v;
    }
    for (int idx = threadIdx.x; idx < n * w; idx += blockDim.x) R[idx] = (idx < ww) ? e[idx] : 0.0;
    __syncthreads();
    if (!sm_lu(F, piv, n, &flag)) {
        if (threadIdx.x == 0) a.status[item] = 2;
        return;
    }
    sm_lu_solve(F, piv, R, n, w);
    __syncthreads();
    double* o = a.out + (size_t)item * ww;
    for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
        const int r = idx / w, c = idx % w;
        double s = 0.0, t = 0.0;
        for (int k = 0; k < w; ++k) {
            s = fma(e[k * w + r], R[k * w + c], s);
            t = fma(e[k * w + c], R[k * w + r], t);
        }
        o[idx] = 0.5 * (s + t);
    }
    if (threadIdx.x == 0) a.status[item] = 0;
}

}  // namespace sfw

using namespace sfw;

// form 0 (tridiag): A = diag blocks [n_models][L][w][w], B = off blocks [n_models][L-1][w][w],
// E = entry blocks [n_models][w][w]; form 1 (chain): A = gammas, B = gamma_hats ([n_models][L][w][w]).
// Items: (model index, omega).  HOST arrays in and out; out [n_items][w][w], status [n_items]
// (0 ok, 2 singular).  Replaces ntd_tridiag / ntd_chain per (model, omega) (ntd.py:101-185).
extern "C" int sfw_ntd_batch(int form, int n_models, int L, int w, const double* A, const double* B, const double* E,
                             int n_items, const int* item_model, const double* item_omega, double* out, int* status,
                             char* errbuf, int errlen) {
    if (form != 0 && form != 1) return fail(SFW_ECONFIG, "form must be 0 (tridiag) or 1 (chain)", errbuf, errlen);
    if (L < 1 || w < 1 || n_items < 0 || n_models < 1) return fail(SFW_ECONFIG, "bad ntd batch shape", errbuf, errlen);
    if (n_items == 0) return 0;
    for (int i = 0; i < n_items; ++i)
        if (item_model[i] < 0 || item_model[i] >= n_models)
            return fail(SFW_ECONFIG, "item model index out of range", errbuf, errlen);
    const size_t ww = (size_t)w * w;
    const size_t na = (size_t)n_models * L * ww;
    const size_t nb = form == 0 ? (size_t)n_models * (L > 1 ? L - 1 : 1) * ww : na;
    double *dA = nullptr, *dB = nullptr, *dE = nullptr, *dom = nullptr, *dout = nullptr;
    int *dmod = nullptr, *dst = nullptr;
    auto cleanup = [&]() {
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dE);
        cudaFree(dom);
        cudaFree(dout);
        cudaFree(dmod);
        cudaFree(dst);
    };
    SFW_CUDA_TRY(cudaMalloc(&dA, na * 8));
    SFW_CUDA_TRY(cudaMalloc(&dB, nb * 8));
    SFW_CUDA_TRY(cudaMalloc(&dE, (form == 0 ? (size_t)n_models * ww : 1) * 8));
    SFW_CUDA_TRY(cudaMalloc(&dom, n_items * 8));
    SFW_CUDA_TRY(cudaMalloc(&dout, (size_t)n_items * ww * 8));
    SFW_CUDA_TRY(cudaMalloc(&dmod, n_items * 4));
    SFW_CUDA_TRY(cudaMalloc(&dst, n_items * 4));
    SFW_CUDA_TRY(sfw_h2d(dA, A, na * 8));
    if (form == 1 || L > 1) SFW_CUDA_TRY(sfw_h2d(dB, B, nb * 8));
    if (form == 0) SFW_CUDA_TRY(sfw_h2d(dE, E, (size_t)n_models * ww * 8));
    SFW_CUDA_TRY(sfw_h2d(dom, item_omega, n_items * 8));
    SFW_CUDA_TRY(sfw_h2d(dmod, item_model, n_items * 4));
    NtdArgs a{form, L, w, dA, dB, dE, dmod, dom, dout, dst};
    const size_t smem = 6 * ww * 8 + (size_t)w * 4 + 16;
    SFW_CUDA_TRY(cudaFuncSetAttribute(k_ntd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_ntd<<<n_items, 256, smem>>>(a);
    SFW_CUDA_TRY(cudaDeviceSynchronize());
    SFW_CUDA_TRY(cudaGetLastError());
    std::vector<int> st(n_items);
    SFW_CUDA_TRY(cudaMemcpy(st.data(), dst, n_items * 4, cudaMemcpyDeviceToHost));
    std::vector<int> fb;
    for (int i = 0; i < n_items; ++i)
        if (st[i] == 1) fb.push_back(i);
    if (!fb.empty()) {
        const size_t n = (size_t)L * w, per = n * n + n * w + n;
        double* work = nullptr;
        int* ditems = nullptr;
        SFW_CUDA_TRY(cudaMalloc(&work, fb.size() * per * 8));
        SFW_CUDA_TRY(cudaMalloc(&ditems, fb.size() * 4));
        SFW_CUDA_TRY(sfw_h2d(ditems, fb.data(), fb.size() * 4));
        k_ntd_assembled<<<(unsigned)fb.size(), 256>>>(a, ditems, work);
        cudaError_t e = cudaDeviceSynchronize();
        cudaFree(work);
        cudaFree(ditems);
        if (e != cudaSuccess) {
            cleanup();
            return fail(SFW_ECUDA, cudaGetErrorString(e), errbuf, errlen);
        }
        SFW_CUDA_TRY(cudaMemcpy(st.data(), dst, n_items * 4, cudaMemcpyDeviceToHost));
    }
    SFW_CUDA_TRY(cudaMemcpy(out, dout, (size_t)n_items * ww * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n_items; ++i) status[i] = st[i];
    cleanup();
    return 0;
}
