// Once-per-run state-space maps of the online stage, on the device:
//   project_source (reference stepper.py:91-128): coeff = (V Q)^T e_s * amp / c_s,
//       first layer block checked and zeroed, out_j = G_j coeff_j
//   make_probe     (reference stepper.py:131-141): w_j = G_j^-T (V Q)[row, blk_j] * c/sqrt(mu)
// One CTA per chain layer; the w x w solve is Gaussian elimination with partial
// pivoting (LAPACK gesv semantics) in shared memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "sfw_common.cuh"

namespace sfw {

// out_j = G_j v_j (kind 0), out_j = G_j^-T v_j (kind 1) or out_j = G_j^-1 v_j (kind 2); v already scaled
__global__ void k_layer_map(const double* __restrict__ G, const double* __restrict__ v, int w, int kind,
                            double* __restrict__ out, int* __restrict__ status) {
    extern __shared__ double sh[];
    const int j = blockIdx.x;
    const double* Gj = G + (size_t)j * w * w;
    const double* vj = v + (size_t)j * w;
    double* oj = out + (size_t)j * w;
    if (kind == 0) {
        for (int i = threadIdx.x; i < w; i += blockDim.x) {
            double s = 0.0;
            for (int k = 0; k < w; ++k) s = fma(Gj[i * w + k], vj[k], s);
            oj[i] = s;
        }
        return;
    }
    double* A = sh;          // w x w : A = G^T
    double* b = sh + w * w;  // w
    __shared__ int piv;
    for (int i = threadIdx.x; i < w * w; i += blockDim.x) {
        const int r = i / w, c = i % w;
        A[i] = (kind == 1) ? Gj[c * w + r] : Gj[i];
    }
    for (int i = threadIdx.x; i < w; i += blockDim.x) b[i] = vj[i];
    __syncthreads();
    for (int c = 0; c < w; ++c) {
        if (threadIdx.x == 0) {
            int pr = c;
            double best = fabs(A[c * w + c]);
            for (int r = c + 1; r < w; ++r)
                if (fabs(A[r * w + c]) > best) {
                    best = fabs(A[r * w + c]);
                    pr = r;
                }
            piv = pr;
            if (best == 0.0) status[j] = 1;
        }
        __syncthreads();
        const int pr = piv;
        if (pr != c) {
            for (int k = threadIdx.x; k < w; k += blockDim.x) {
                const double t = A[c * w + k];
                A[c * w + k] = A[pr * w + k];
                A[pr * w + k] = t;
            }
            if (threadIdx.x == 0) {
                const double t = b[c];
                b[c] = b[pr];
                b[pr] = t;
            }
        }
        __syncthreads();
        for (int r = c + 1 + threadIdx.x; r < w; r += blockDim.x) {
            const double l = A[r * w + c] / A[c * w + c];
            for (int k = c + 1; k < w; ++k) A[r * w + k] -= l * A[c * w + k];
            b[r] -= l * b[c];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        for (int c = w - 1; c >= 0; --c) {
            double s = b[c];
            for (int k = c + 1; k < w; ++k) s -= A[c * w + k] * b[k];
            b[c] = s / A[c * w + c];
        }
        for (int i = 0; i < w; ++i) oj[i] = b[i];
    }
}

// out[k] = sum_n B[n][k] x[n] (B row-major N x K): one thread per column, n ascending
__global__ void k_basis_t(const double* __restrict__ B, const double* __restrict__ x, int N, int K,
                          double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    double s = 0.0;
    for (int n = 0; n < N; ++n) s = fma(B[(size_t)n * K + k], x[n], s);
    out[k] = s;
}

// out[n] = sum_k B[n][k] c[k]: one warp per row, lane-strided partials, fixed-order butterfly
__global__ void k_basis_n(const double* __restrict__ B, const double* __restrict__ c, int N, int K,
                          double* __restrict__ out) {
    const int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (n >= N) return;
    double s = 0.0;
    for (int k = lane; k < K; k += 32) s = fma(B[(size_t)n * K + k], c[k], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[n] = s;
}

__global__ void k_scale_vec(const double* __restrict__ x, long long n, double s, double* __restrict__ y) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = x[i] * s;
}

__global__ void k_norm_pair(const double* __restrict__ x, long long n, int w, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (long long i = 0; i < n; ++i) {
            a += x[i] * x[i];
            if (i < w) b += x[i] * x[i];
        }
        out[0] = sqrt(a);
        out[1] = sqrt(b);
    }
}

__global__ void k_zero_head(double* __restrict__ x, int w) {
    for (int i = threadIdx.x; i < w; i += blockDim.x) x[i] = 0.0;
}

}  // namespace sfw

using namespace sfw;

static int maps_common(int L, int w, const double* G, const double* row, double scale, int kind, double* out,
                       double* norms, char* errbuf, int errlen) {
    const size_t K = (size_t)L * w;
    double *dG = nullptr, *dv = nullptr, *dc = nullptr, *dout = nullptr, *dn = nullptr;
    int* dst = nullptr;
    int rc = 0;
    auto cleanup = [&]() {
        cudaFree(dG);
        cudaFree(dv);
        cudaFree(dc);
        cudaFree(dout);
        cudaFree(dn);
        cudaFree(dst);
    };
    if (dalloc(&dG, K * w, errbuf, errlen) || dalloc(&dv, K, errbuf, errlen) || dalloc(&dc, K, errbuf, errlen) ||
        dalloc(&dout, K, errbuf, errlen) || dalloc(&dn, 2, errbuf, errlen) || dalloc(&dst, L, errbuf, errlen)) {
        cleanup();
        return SFW_ECUDA;
    }
    sfw_h2d(dG, G, K * w * 8);
    sfw_h2d(dv, row, K * 8);
    cudaMemset(dst, 0, L * sizeof(int));
    if (kind == 0) {
        // coeff = row * (amp / c); leak check on the first block; zero it; apply G_j
        k_scale_vec<<<8, 256>>>(dv, (long long)K, scale, dc);
        k_norm_pair<<<1, 32>>>(dc, (long long)K, w, dn);
        cudaMemcpy(norms, dn, 16, cudaMemcpyDeviceToHost);
        k_zero_head<<<1, 256>>>(dc, w);
        k_layer_map<<<L, 128>>>(dG, dc, w, 0, dout, dst);
        cudaMemcpy(out, dout, K * 8, cudaMemcpyDeviceToHost);
    } else {
        const size_t sm = (size_t)(w * w + w) * 8;
        cudaFuncSetAttribute(k_layer_map, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_layer_map<<<L, 128, sm>>>(dG, dv, w, 1, dc, dst);
        k_scale_vec<<<8, 256>>>(dc, (long long)K, scale, dout);
        cudaMemcpy(out, dout, K * 8, cudaMemcpyDeviceToHost);
        std::vector<int> st(L);
        cudaMemcpy(st.data(), dst, L * sizeof(int), cudaMemcpyDeviceToHost);
        for (int j = 0; j < L; ++j)
            if (st[j]) rc = fail(SFW_ENUMERICAL, "singular chain scale matrix in make_probe", errbuf, errlen);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = fail(SFW_ECUDA, cudaGetErrorString(e), errbuf, errlen);
    cleanup();
    return rc;
}

extern "C" int sfw_source_vector(int L, int w, const double* scales, const double* basis_row, double scale,
                                 double* out, double* norms, char* errbuf, int errlen) {
    return maps_common(L, w, scales, basis_row, scale, 0, out, norms, errbuf, errlen);
}

extern "C" int sfw_probe_weights(int L, int w, const double* scales, const double* basis_row, double scale,
                                 double* out, char* errbuf, int errlen) {
    return maps_common(L, w, scales, basis_row, scale, 1, out, nullptr, errbuf, errlen);
}

// project_state / state_to_nodes (reference rom.py:437-459): basis HOST N x K row-major (V Q as
// SubdomainModel.basis stores it), scales HOST L x w x w; dir 0: x = node field (N) -> out (K),
// out_j = G_j (B^T x)_j; dir 1: x = chain state (K) -> out (N) = B (G_j^-1 x_j)_j.
static int state_map(int dir, int N, int L, int w, const double* basis, const double* scales, const double* x,
                     double* out, char* errbuf, int errlen) {
    if (N < 1 || L < 1 || w < 1 || !basis || !scales || !x || !out)
        return fail(SFW_ECONFIG, "state map: bad sizes or NULL arrays", errbuf, errlen);
    const int K = L * w;
    double *dB = nullptr, *dG = nullptr, *dx = nullptr, *dc = nullptr, *dout = nullptr;
    int* dst = nullptr;
    auto cleanup = [&]() {
        cudaFree(dB);
        cudaFree(dG);
        cudaFree(dx);
        cudaFree(dc);
        cudaFree(dout);
        cudaFree(dst);
    };
    if (dalloc(&dB, (size_t)N * K, errbuf, errlen) || dalloc(&dG, (size_t)K * w, errbuf, errlen) ||
        dalloc(&dx, (size_t)std::max(N, K), errbuf, errlen) || dalloc(&dc, (size_t)K, errbuf, errlen) ||
        dalloc(&dout, (size_t)std::max(N, K), errbuf, errlen) || dalloc(&dst, (size_t)L, errbuf, errlen)) {
        cleanup();
        return SFW_ECUDA;
    }
    sfw_h2d(dB, basis, (size_t)N * K * 8);
    sfw_h2d(dG, scales, (size_t)K * w * 8);
    sfw_h2d(dx, x, (size_t)(dir == 0 ? N : K) * 8);
    cudaMemset(dst, 0, L * sizeof(int));
    int rc = 0;
    if (dir == 0) {
        k_basis_t<<<(K + 127) / 128, 128>>>(dB, dx, N, K, dc);
        k_layer_map<<<L, 128>>>(dG, dc, w, 0, dout, dst);
        cudaMemcpy(out, dout, (size_t)K * 8, cudaMemcpyDeviceToHost);
    } else {
        const size_t sm = (size_t)(w * w + w) * 8;
        cudaFuncSetAttribute(k_layer_map, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_layer_map<<<L, 128, sm>>>(dG, dx, w, 2, dc, dst);
        k_basis_n<<<(N * 32 + 255) / 256, 256>>>(dB, dc, N, K, dout);
        cudaMemcpy(out, dout, (size_t)N * 8, cudaMemcpyDeviceToHost);
        std::vector<int> st(L);
        cudaMemcpy(st.data(), dst, L * sizeof(int), cudaMemcpyDeviceToHost);
        for (int j = 0; j < L; ++j)
            if (st[j]) rc = fail(SFW_ENUMERICAL, "singular chain scale matrix in state_to_nodes", errbuf, errlen);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = fail(SFW_ECUDA, cudaGetErrorString(e), errbuf, errlen);
    cleanup();
    return rc;
}

extern "C" int sfw_project_state(int N, int L, int w, const double* basis, const double* scales, const double* x,
                                 double* out, char* errbuf, int errlen) {
    return state_map(0, N, L, w, basis, scales, x, out, errbuf, errlen);
}

extern "C" int sfw_state_to_nodes(int N, int L, int w, const double* basis, const double* scales, const double* u,
                                  double* out, char* errbuf, int errlen) {
    return state_map(1, N, L, w, basis, scales, u, out, errbuf, errlen);
}
