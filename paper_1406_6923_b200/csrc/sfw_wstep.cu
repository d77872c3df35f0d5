// fp32 W-form stepping (BASELINE config 5 fp32 variant).
//
// The reference U-form (stepper.py:291-309) rounded to fp32 diverges at m=9,
// k=8.  With U_j = G_j W_j the chain becomes the Lanczos block
// tridiagonal operator of rom.py:202-262:
//     W_j'' = A_j W_j + B_j^T W_{j+1} + B_{j-1} W_{j-1}        (0-based; B_j couples j, j+1)
// with A_j = -G_j^T (Gamma_j + Gamma_{j-1}) G_j, B_j = G_{j+1}^T Gamma_j G_j, and
// the interface mass of stepper.py:204-210 becomes exactly 1/2 (Gamma-hat_1 = I).
// It is the same ROM to rounding (fp64 W vs U form: 2.5e-13 at m4k4) and stable
// in fp32 (1e-6 vs the fp64 reference).  Blocks are half the bytes of fp64 and
// each of A_j (symmetric) and B_j (triangular, stored as B_j^T lower-packed) is
// streamed once per step:
//   round 1: item (s, j): p_j = A_j W_j + B_j^T W_{j+1};  c_{j+1} = B_j W_j
//   round 2: layers j >= 1: W'' = p_j + c_j (+ source), leapfrog
//   round 3: layer 0: shared faces 1/2 (p_0 + p_0'), exterior p_0, leapfrog, probes
// Layer-0 partials double as the face mailbox (double-buffered by step parity).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sfw_common.cuh"
#include "sfw_linalg.cuh"
#include "sfw_step_internal.cuh"

namespace sfw {

namespace wf {
__host__ __device__ constexpr int tri_count(int m) { return m * (m + 1) / 2; }
__host__ __device__ constexpr int packed_len(int m) { return 15 * m * m + 6 * tri_count(m); }
__host__ __device__ constexpr int packed_stride32(int m) { return (packed_len(m) + 3) & ~3; }
__host__ __device__ constexpr int off_I(int t) { return t < 1 ? 1 : t < 3 ? 2 : t < 6 ? 3 : t < 10 ? 4 : 5; }
__host__ __device__ constexpr int off_K(int t) { return t - off_I(t) * (off_I(t) - 1) / 2; }
__host__ __device__ constexpr int off_tile(int I, int K) { return I * (I - 1) / 2 + K; }

// same 6-group lower-packed layout as the fp64 stepper (sfw_step.cu packed_pos)
__host__ __device__ inline int packed_pos(int m, int row, int col) {
    int I = row / m, K = col / m, r = row % m, c = col % m;
    if (I != K) {
        const int t = off_tile(I, K);
        const int q = (c - r + m) % m;
        return (q * m + r) * 15 + t;
    }
    const int d = r - c;
    int e = 0;
    for (int dd = 0; dd < d; ++dd) e += m - dd;
    e += c;
    return 15 * m * m + e * 6 + I;
}
}  // namespace wf

// offsets of the partials summed into each output row (conflict-free layout slot*21 + tile)
template <int M>
struct WRed {
    static constexpr int W = 6 * M, EPL = (W + 31) / 32;
    int sym[EPL][6];  // symmetric product: 6 terms (as sfw_step.cu RedOff)
    int lo[EPL][6];   // L x   : rows R: tiles (R,K<=R) row partials, -1 padded
    int up[EPL][6];   // L^T x': rows K: tiles (I>=K,K) column partials, -1 padded
    __device__ __forceinline__ explicit WRed(int lane) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            const int i = lane + 32 * e;
            const int R = i < W ? i / M : 0, r = i < W ? i % M : 0;
#pragma unroll
            for (int t = 0; t < 6; ++t) {
                sym[e][t] = (t < R) ? r * 21 + wf::off_tile(R, t)
                                    : (t == R) ? r * 21 + 15 + R : (M + r) * 21 + wf::off_tile(t, R);
                lo[e][t] = (t < R) ? r * 21 + wf::off_tile(R, t) : (t == R) ? r * 21 + 15 + R : -1;
                up[e][t] = (t == R) ? (M + r) * 21 + 15 + R : (t > R) ? (M + r) * 21 + wf::off_tile(t, R) : -1;
            }
        }
    }
};

// y = A x, A symmetric lower-packed (fp32, one warp)
template <int M>
__device__ __forceinline__ void wsym(const float* __restrict__ blk, const float* x, float* part, float* y, int lane,
                                     const WRed<M>& ro) {
    constexpr int W = 6 * M;
    if (lane < 15) {
        const int I = wf::off_I(lane), K = wf::off_K(lane);
        float xk[M], xi[M], P[M], Q[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            xk[i] = x[K * M + i];
            xi[i] = x[I * M + i];
            P[i] = Q[i] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < M * M; ++e) {
            const int r = e % M, c = (e / M + r) % M;
            const float a = blk[e * 15 + lane];
            P[r] = fmaf(a, xk[c], P[r]);
            Q[c] = fmaf(a, xi[r], Q[c]);
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
            part[i * 21 + lane] = P[i];
            part[(M + i) * 21 + lane] = Q[i];
        }
    }
    if (lane < 6) {
        float xi[M], P[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            xi[i] = x[lane * M + i];
            P[i] = 0.f;
        }
        const float* b = blk + 15 * M * M + lane;
#pragma unroll
        for (int d = 0; d < M; ++d)
#pragma unroll
            for (int r = d; r < M; ++r) {
                const int c = r - d;
                const float a = b[(d * M - d * (d - 1) / 2 + c) * 6];
                P[r] = fmaf(a, xi[c], P[r]);
                if (d != 0) P[c] = fmaf(a, xi[r], P[c]);
            }
#pragma unroll
        for (int i = 0; i < M; ++i) part[i * 21 + 15 + lane] = P[i];
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < WRed<M>::EPL; ++e) {
        const int i = lane + 32 * e;
        if (i < W) {
            float s = part[ro.sym[e][0]];
#pragma unroll
            for (int t = 1; t < 6; ++t) s += part[ro.sym[e][t]];
            y[i] = s;
        }
    }
    __syncwarp();
}

// y1 = Lo x (Lo lower-packed incl. diagonal), y2 = Lo^T x2   (one warp, one pass over Lo)
template <int M>
__device__ __forceinline__ void wtri2(const float* __restrict__ blk, const float* x, const float* x2, float* part,
                                      float* y1, float* y2, int lane, const WRed<M>& ro) {
    constexpr int W = 6 * M;
    if (lane < 15) {
        const int I = wf::off_I(lane), K = wf::off_K(lane);
        float xk[M], xi[M], P[M], Q[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            xk[i] = x[K * M + i];
            xi[i] = x2[I * M + i];
            P[i] = Q[i] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < M * M; ++e) {
            const int r = e % M, c = (e / M + r) % M;
            const float a = blk[e * 15 + lane];
            P[r] = fmaf(a, xk[c], P[r]);
            Q[c] = fmaf(a, xi[r], Q[c]);
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
            part[i * 21 + lane] = P[i];
            part[(M + i) * 21 + lane] = Q[i];
        }
    }
    if (lane < 6) {
        float xa[M], xb[M], P[M], Q[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            xa[i] = x[lane * M + i];
            xb[i] = x2[lane * M + i];
            P[i] = Q[i] = 0.f;
        }
        const float* b = blk + 15 * M * M + lane;
#pragma unroll
        for (int d = 0; d < M; ++d)
#pragma unroll
            for (int r = d; r < M; ++r) {
                const int c = r - d;
                const float a = b[(d * M - d * (d - 1) / 2 + c) * 6];
                P[r] = fmaf(a, xa[c], P[r]);
                Q[c] = fmaf(a, xb[r], Q[c]);
            }
#pragma unroll
        for (int i = 0; i < M; ++i) {
            part[i * 21 + 15 + lane] = P[i];
            part[(M + i) * 21 + 15 + lane] = Q[i];
        }
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < WRed<M>::EPL; ++e) {
        const int i = lane + 32 * e;
        if (i < W) {
            float s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int t = 0; t < 6; ++t) {
                if (ro.lo[e][t] >= 0) s1 += part[ro.lo[e][t]];
                if (ro.up[e][t] >= 0) s2 += part[ro.up[e][t]];
            }
            y1[i] = s1;
            y2[i] = s2;
        }
    }
    __syncwarp();
}

struct WParams {
    int n_sub, L, BS, n_steps, record_every, n_probe, ftab_stride, mode;  // mode 0 step, 1 init
    double dt;
    float dt2, half;
    const float* coef;      // [n_sub][2L-1][BS]: A_0, B_0, A_1, B_1, ..., A_{L-1}
    float* W0;
    float* W1;
    const float* V0;        // init velocity (W-form) or null
    float* P;               // [2][n_sub][K] row partials (layer 0 = face mailbox)
    float* Cc;              // [n_sub][K] carries B_{j-1} W_{j-1}
    const int* cta_sub_ptr;
    const int* nbr;
    const int* src_ptr;
    const int* src_ids;
    const float* src_vec;   // W-form source vectors
    const long long* src_voff;
    const float* ftab;      // [n_src][ftab_stride] profile values
    const int* prb_ptr;
    const int* prb_ids;
    const int* prb_tap;
    const float* prb_w;     // W-form probe weights
    const long long* prb_woff;
    double* rows;
    double* sub_norm;
    double* sqs;            // [n_sub][L]
    double* norm_part;
    unsigned int* flags;
    const int* ncta_ptr;
    const int* ncta;
};

__device__ __forceinline__ float wforce(const WParams& p, int s, long long idx, int k, float acc) {
    const int a = p.src_ptr[s], b = p.src_ptr[s + 1];
    for (int q = a; q < b; ++q) {
        const int src = p.src_ids[q];
        acc = fmaf(p.src_vec[p.src_voff[src] + idx], p.ftab[(size_t)src * p.ftab_stride + k], acc);
    }
    return acc;
}

__device__ __forceinline__ float wleap(int mode, float u, float uo, float v, float tot, float dt, float dt2,
                                       float half) {
    if (mode == 0) return fmaf(dt2, tot, 2.f * u - uo);
    return fmaf(half, tot, u - dt * v);
}

template <int M, int NW, int NS>
__global__ void __launch_bounds__(NW * 32, 1) k_wstep(const WParams p) {
    constexpr int W = 6 * M;
    constexpr int EPL = (W + 31) / 32;
    constexpr int WK = 4 * W + 21 * 2 * M;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const WRed<M> ro(lane);
    const int BS = p.BS, L = p.L;
    const long long K = (long long)L * W;
    float* stages = reinterpret_cast<float*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + (size_t)NW * NS * BS);
    float* wk = reinterpret_cast<float*>(bars + NW * NS) + (size_t)warp * WK;
    float* xa = wk;         // W_j
    float* xb = xa + W;     // W_{j+1}
    float* y1 = xb + W;
    float* y2 = y1 + W;
    float* part = y2 + W;
    float* my_stage = stages + (size_t)warp * NS * BS;
    uint64_t* my_bar = bars + warp * NS;
    if (lane == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&my_bar[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int s0 = p.cta_sub_ptr[blockIdx.x], s1 = p.cta_sub_ptr[blockIdx.x + 1];
    const int nit = (s1 - s0) * L;
    const int n1 = nit > warp ? (nit - warp + NW - 1) / NW : 0;
    const int n_iter = p.mode == 0 ? p.n_steps : 1;
    // blocks per step for this warp: its items, 2 blocks each except the last layer (1)
    int per = 0;
    for (int t = 0; t < n1; ++t) per += ((warp + t * NW) % L == L - 1) ? 1 : 2;
    const int total = per * n_iter;
    const uint64_t pol = l2_policy_evict_first();
    const uint32_t bytes = (uint32_t)BS * 4u;
    int issued = 0, consumed = 0, pr_t = 0, pr_b = 0;  // producer: item index, block within item
    auto issue = [&]() {
        if (lane == 0)
            while (issued < total && issued < consumed + NS) {
                const int q = warp + pr_t * NW;
                const int s = s0 + q / L, j = q % L;
                const long long blk = (long long)s * (2 * L - 1) + 2 * j + pr_b;
                const int st = issued % NS;
                fence_proxy_async();
                mbar_arrive_expect_tx(&my_bar[st], bytes);
                bulk_g2s(my_stage + (size_t)st * BS, p.coef + blk * BS, bytes, &my_bar[st], pol);
                ++issued;
                if (pr_b == 0 && j < L - 1) {
                    pr_b = 1;
                } else {
                    pr_b = 0;
                    if (++pr_t == n1) pr_t = 0;
                }
            }
    };
    auto acquire = [&]() -> const float* {
        const int st = consumed % NS;
        mbar_wait(&my_bar[st], (uint32_t)((consumed / NS) & 1));
        return my_stage + (size_t)st * BS;
    };
    auto release = [&]() {
        __syncwarp();
        ++consumed;
        issue();
    };
    issue();
    const float dt = (float)p.dt, dt2 = p.dt2, half = p.half;

    for (int k = 1; k <= n_iter; ++k) {
        const int par = k & 1;
        const int cb = (k - 1) & 1;
        const float* Wc = cb ? p.W1 : p.W0;
        float* Wn = cb ? p.W0 : p.W1;
        float* Pp = p.P + (size_t)par * p.n_sub * K;
        const int kk = k - 1;
        // ---------------- round 1: row partials and carries ----------------------
        {
            float na[EPL], nb[EPL];  // next item's W_j, W_{j+1} (register prefetch)
            auto load = [&](int t) {
                const int q = warp + t * NW;
                const int s = s0 + q / L, j = q % L;
                const float* w = Wc + (size_t)s * K + (size_t)j * W;
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    const int i = lane + 32 * e;
                    na[e] = (i < W) ? w[i] : 0.f;
                    nb[e] = (i < W && j + 1 < L) ? w[W + i] : 0.f;
                }
            };
            if (n1 > 0) load(0);
            for (int t = 0; t < n1; ++t) {
                const int q = warp + t * NW;
                const int s = s0 + q / L, j = q % L;
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    const int i = lane + 32 * e;
                    if (i < W) {
                        xa[i] = na[e];
                        xb[i] = nb[e];
                    }
                }
                if (t + 1 < n1) load(t + 1);
                __syncwarp();
                wsym<M>(acquire(), xa, part, y1, lane, ro);
                release();
                float* pj = Pp + (size_t)s * K + (size_t)j * W;
                if (j + 1 < L) {
                    for (int i = lane; i < W; i += 32) y2[i] = y1[i];
                    __syncwarp();
                    wtri2<M>(acquire(), xb, xa, part, y1, xb, lane, ro);
                    release();
                    float* cj = p.Cc + (size_t)s * K + (size_t)(j + 1) * W;
                    for (int i = lane; i < W; i += 32) {
                        pj[i] = y2[i] + y1[i];
                        cj[i] = xb[i];
                    }
                } else {
                    for (int i = lane; i < W; i += 32) pj[i] = y1[i];
                }
                __syncwarp();
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) flag_publish(p.flags, (unsigned int)k);
        double sq = 0.0;  // this thread's share of |W_next|^2 (fixed element order)
        // ---------------- round 2: interior layers, CTA-wide elementwise ----------
        {
            const int per_sub = (L - 1) * W;
            const int nel = (s1 - s0) * per_sub;
            constexpr int U = 4;
            for (int base = threadIdx.x; base < nel; base += U * NW * 32) {
                float pv[U], cv[U], wc[U], wo[U], vv[U];
                size_t off[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int idx = base + u * NW * 32;
                    if (idx < nel) {
                        const int sl = idx / per_sub, r = idx % per_sub;
                        off[u] = (size_t)(s0 + sl) * K + W + r;
                        pv[u] = Pp[off[u]];
                        cv[u] = p.Cc[off[u]];
                        wc[u] = Wc[off[u]];
                        wo[u] = (p.mode == 0) ? Wn[off[u]] : 0.f;
                        vv[u] = (p.mode == 1 && p.V0) ? p.V0[off[u]] : 0.f;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int idx = base + u * NW * 32;
                    if (idx < nel) {
                        const int sl = idx / per_sub, r = idx % per_sub;
                        const int s = s0 + sl;
                        const float tot = wforce(p, s, (long long)W + r, kk, pv[u] + cv[u]);
                        const float un = wleap(p.mode, wc[u], wo[u], vv[u], tot, dt, dt2, half);
                        Wn[off[u]] = un;
                        sq = fma((double)un, (double)un, sq);
                    }
                }
            }
        }
        __syncthreads();
        if (warp == 0)
            flags_wait(p.flags, p.ncta + p.ncta_ptr[blockIdx.x], p.ncta_ptr[blockIdx.x + 1] - p.ncta_ptr[blockIdx.x],
                       (unsigned int)k, lane);
        __syncthreads();
        // ---------------- round 3: layer 0 + faces, probes ------------------------
        for (int s = s0 + warp; s < s1; s += NW) {
            const size_t o = (size_t)s * K;
            for (int i = lane; i < W; i += 32) {
                const int f = i / M;
                const int nbs = p.nbr[s * 6 + f];
                float a = Pp[o + i];
                if (nbs >= 0) a = 0.5f * (a + Pp[(size_t)nbs * K + (f ^ 1) * M + i % M]);
                const float tot = wforce(p, s, i, kk, a);
                const float v = (p.mode == 1 && p.V0) ? p.V0[o + i] : 0.f;
                const float un = wleap(p.mode, Wc[o + i], (p.mode == 0) ? Wn[o + i] : 0.f, v, tot, dt, dt2, half);
                Wn[o + i] = un;
                sq = fma((double)un, (double)un, sq);
            }
        }
        // per-CTA |W|^2 partial (fixed-order block reduction)
        {
            double v = warp_sum(sq);
            __shared__ double wred[32];
            if (lane == 0) wred[warp] = v;
            __syncthreads();
            if (threadIdx.x == 0 && p.mode == 0) {
                double tsum = 0.0;
                for (int i = 0; i < NW; ++i) tsum += wred[i];
                p.norm_part[(size_t)kk * gridDim.x + blockIdx.x] = tsum;
            }
        }
        // probes (all layers written by now)
        const bool rec = (p.mode == 1) || (k % p.record_every == 0);
        if (rec && p.rows) {
            const long long row = (p.mode == 1) ? 0 : (k / p.record_every - 1);
            for (int s = s0 + warp; s < s1; s += NW) {
                if (p.prb_ptr[s] == p.prb_ptr[s + 1]) continue;
                const float* U = ((p.mode == 1) ? Wc : Wn) + (size_t)s * K;
                for (int pq = p.prb_ptr[s]; pq < p.prb_ptr[s + 1]; ++pq) {
                    const int pid = p.prb_ids[pq];
                    double val = 0.0;
                    const float* wv = p.prb_w + p.prb_woff[pid];
                    for (long long i = lane; i < K; i += 32) val = fma((double)wv[i], (double)U[i], val);
                    val = warp_sum(val);
                    if (lane == 0) p.rows[row * p.n_probe + pid] = val;
                }
            }
        }
        __syncthreads();
    }
    (void)EPL;
}

// ---------------------------------------------------------------------------
// setup: T blocks from (G, Gamma) in fp64, packed to fp32; vector conversions

// one CTA per (subdomain, layer j): A_j = -G_j^T (Gamma_j + Gamma_{j-1}) G_j and, for j < L-1,
// B_j = G_{j+1}^T Gamma_j G_j stored as B_j^T (lower) -> both packed fp32
__global__ void k_wform_blocks(const double* __restrict__ G, const double* __restrict__ Gam, const int* lay_sub,
                               const int* lay_j, const long long* __restrict__ first_blk, const int* __restrict__ layers,
                               int m, int BS, float* __restrict__ out) {
    extern __shared__ double sm[];
    const int w = 6 * m, ww = w * w;
    double* A = sm;
    double* B = A + ww;
    double* C = B + ww;
    const int q = blockIdx.x;
    const int s = lay_sub[q], j = lay_j[q], L = layers[s];
    const double* Gs = G + first_blk[s];
    const double* Gm = Gam + first_blk[s];
    // C = Gamma_j + Gamma_{j-1}
    for (int i = threadIdx.x; i < ww; i += blockDim.x)
        C[i] = Gm[(size_t)j * ww + i] + (j > 0 ? Gm[(size_t)(j - 1) * ww + i] : 0.0);
    __syncthreads();
    sm_matmul(C, false, Gs + (size_t)j * ww, false, B, w);   // B = C G_j
    sm_matmul(Gs + (size_t)j * ww, true, B, false, A, w);    // A = G_j^T C G_j
    const long long blk = (long long)s * (2 * L - 1) + 2 * j;  // uniform layer count (checked at setup)
    float* oa = out + blk * BS;
    for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
        const int r = idx / w, c = idx % w;
        if (r >= c) oa[wf::packed_pos(m, r, c)] = (float)(-0.5 * (A[r * w + c] + A[c * w + r]));
    }
    if (j + 1 < L) {
        __syncthreads();
        sm_matmul(Gm + (size_t)j * ww, false, Gs + (size_t)j * ww, false, B, w);       // B = Gamma_j G_j
        sm_matmul(Gs + (size_t)(j + 1) * ww, true, B, false, C, w);                   // C = G_{j+1}^T Gamma_j G_j
        float* ob = out + (blk + 1) * BS;
        for (int idx = threadIdx.x; idx < ww; idx += blockDim.x) {
            const int r = idx / w, c = idx % w;
            if (r >= c) ob[wf::packed_pos(m, r, c)] = (float)C[c * w + r];  // (B_j)^T lower: element (r,c) = B_j[c][r]
        }
    }
}

// per (vector, layer) CTA: mode 0: out = G^-1 v ; mode 1: out = G^T v ; mode 2: out = G v   (fp64)
__global__ void k_layer_apply(const double* __restrict__ G, const long long* __restrict__ first_blk,
                              const int* __restrict__ vsub, const long long* __restrict__ voff,
                              const int* __restrict__ lay_of_vec, int w, int mode, const double* __restrict__ in,
                              double* __restrict__ out) {
    extern __shared__ double sm[];
    const int v = lay_of_vec[2 * blockIdx.x], j = lay_of_vec[2 * blockIdx.x + 1];
    const int s = vsub[v];
    const double* Gj = G + first_blk[s] + (size_t)j * w * w;
    const double* x = in + voff[v] + (size_t)j * w;
    double* y = out + voff[v] + (size_t)j * w;
    if (mode != 0) {
        for (int i = threadIdx.x; i < w; i += blockDim.x) {
            double acc = 0.0;
            for (int c = 0; c < w; ++c) acc = fma(mode == 1 ? Gj[c * w + i] : Gj[i * w + c], x[c], acc);
            y[i] = acc;
        }
        return;
    }
    double* A = sm;
    double* b = A + w * w;
    int* piv = reinterpret_cast<int*>(b + w);
    __shared__ int flag;
    for (int i = threadIdx.x; i < w * w; i += blockDim.x) A[i] = Gj[i];
    for (int i = threadIdx.x; i < w; i += blockDim.x) b[i] = x[i];
    __syncthreads();
    sm_lu(A, piv, w, &flag);
    sm_lu_solve(A, piv, b, w, 1);
    for (int i = threadIdx.x; i < w; i += blockDim.x) y[i] = b[i];
}

__global__ void k_d2f(const double* __restrict__ a, float* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}
__global__ void k_f2d(const float* __restrict__ a, double* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        b[i] = (double)a[i];
}

}  // namespace sfw

using namespace sfw;

namespace {
struct WState {
    int BS = 0, nw = 0, ns = 0, smem = 0;
    const void* fn = nullptr;
    float *coef = nullptr, *W[2] = {nullptr, nullptr}, *V0 = nullptr, *P = nullptr, *Cc = nullptr;
    float *src = nullptr, *prb = nullptr, *ftab = nullptr;
    long long ftab_cap = 0;
    double *sqs = nullptr, *d_tmp = nullptr, *d_tmp2 = nullptr;
    long long* first_blk = nullptr;
    int cur = 0;
};
}  // namespace

// the W-form state hangs off the stepper handle (opaque pointer kept in a side table)
#include <map>
static std::map<sfw_stepper*, WState*> g_wf;

static int wf_vectors(sfw_stepper* h, WState* ws, int nvec, const int* vsub_h, const long long* voff_h, long long n,
                      int mode, const double* in_host, double* out_host, char* errbuf, int errlen) {
    // apply per-layer G maps to nvec state-space vectors on the device
    std::vector<int> lv;
    for (int v = 0; v < nvec; ++v)
        for (int j = 0; j < h->layers[vsub_h[v]]; ++j) {
            lv.push_back(v);
            lv.push_back(j);
        }
    int *d_vs = nullptr, *d_lv = nullptr;
    long long* d_vo = nullptr;
    double *d_in = nullptr, *d_out = nullptr;
    int rc = 0;
    std::vector<int> vs(vsub_h, vsub_h + nvec);
    std::vector<long long> vo(voff_h, voff_h + nvec);
    if ((rc = upload(&d_vs, vs, errbuf, errlen)) || (rc = upload(&d_vo, vo, errbuf, errlen)) ||
        (rc = upload(&d_lv, lv, errbuf, errlen)) || (rc = dalloc(&d_in, n, errbuf, errlen)) ||
        (rc = dalloc(&d_out, n, errbuf, errlen)))
        return rc;
    cudaMemcpy(d_in, in_host, n * 8, cudaMemcpyHostToDevice);
    const int w = h->W;
    const size_t sm = (size_t)(w * w + w) * 8 + w * 4 + 16;
    cudaFuncSetAttribute(k_layer_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (!lv.empty())
        k_layer_apply<<<(unsigned)(lv.size() / 2), 128, sm, h->stream>>>(h->scales, ws->first_blk, d_vs, d_vo, d_lv, w,
                                                                       mode, d_in, d_out);
    cudaStreamSynchronize(h->stream);
    cudaMemcpy(out_host, d_out, n * 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    cudaFree(d_vs);
    cudaFree(d_vo);
    cudaFree(d_lv);
    cudaFree(d_in);
    cudaFree(d_out);
    if (e != cudaSuccess) return fail(SFW_ECUDA, cudaGetErrorString(e), errbuf, errlen);
    return 0;
}

// Switch a stepper to fp32 W-form (requires the scales G_j at creation).
// src_vec / probe weights of the handle are converted from U-form on the device.
extern "C" int sfw_wform_setup(sfw_stepper* h, char* errbuf, int errlen) {
    if (!h->scales) return fail(SFW_ECONFIG, "fp32 W-form stepping needs the models' scales (G_j)", errbuf, errlen);
    if (!h->uniform) return fail(SFW_ECONFIG, "fp32 W-form stepping needs one layer count", errbuf, errlen);
    if (h->m != 4 && h->m != 9 && h->m != 1)
        return fail(SFW_ECONFIG, "fp32 W-form stepping supports m = 1, 4, 9", errbuf, errlen);
    if (g_wf.count(h)) return 0;
    auto* ws = new WState();
    const int m = h->m, w = h->W, n = h->n_sub, L = h->L;
    ws->BS = wf::packed_stride32(m);
    const long long nb = (long long)n * (2 * L - 1);
    const long long K = (long long)L * w;
    int rc = 0;
    std::vector<long long> fb(n);
    for (int s = 0; s < n; ++s) fb[s] = (long long)s * L * w * w;
    std::vector<int> ls, lj;
    for (int s = 0; s < n; ++s)
        for (int j = 0; j < L; ++j) {
            ls.push_back(s);
            lj.push_back(j);
        }
    int *d_ls = nullptr, *d_lj = nullptr;
    if ((rc = dalloc(&ws->coef, (size_t)nb * ws->BS, errbuf, errlen)) || (rc = upload(&ws->first_blk, fb, errbuf, errlen)) ||
        (rc = upload(&d_ls, ls, errbuf, errlen)) || (rc = upload(&d_lj, lj, errbuf, errlen)) ||
        (rc = dalloc(&ws->W[0], (size_t)n * K, errbuf, errlen)) || (rc = dalloc(&ws->W[1], (size_t)n * K, errbuf, errlen)) ||
        (rc = dalloc(&ws->P, (size_t)2 * n * K, errbuf, errlen)) || (rc = dalloc(&ws->Cc, (size_t)n * K, errbuf, errlen)) ||
        (rc = dalloc(&ws->sqs, (size_t)n * L, errbuf, errlen)))
        return rc;
    cudaMemsetAsync(ws->coef, 0, (size_t)nb * ws->BS * 4, h->stream);
    cudaMemsetAsync(ws->P, 0, (size_t)2 * n * K * 4, h->stream);
    const size_t sm = (size_t)3 * w * w * 8;
    SFW_CUDA_TRY(cudaFuncSetAttribute(k_wform_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_wform_blocks<<<(unsigned)ls.size(), 256, sm, h->stream>>>(h->scales, h->gam_dense, d_ls, d_lj, ws->first_blk,
                                                                h->d_layers, m, ws->BS, ws->coef);
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    cudaFree(d_ls);
    cudaFree(d_lj);
    // kernel variant
    const char* env_nw = getenv("SFW_WSTEP_NW");
    const int want = env_nw ? atoi(env_nw) : 12;
    if (m == 9 && want == 16) {
        ws->nw = 16;
        ws->ns = 2;
        ws->fn = (const void*)k_wstep<9, 16, 2>;
    } else if (m == 9 && want == 12) {
        ws->nw = 12;
        ws->ns = 2;
        ws->fn = (const void*)k_wstep<9, 12, 2>;
    } else if (m == 9) {
        ws->nw = 8;
        ws->ns = 4;
        ws->fn = (const void*)k_wstep<9, 8, 4>;
    } else if (m == 4) {
        ws->nw = 16;
        ws->ns = 4;
        ws->fn = (const void*)k_wstep<4, 16, 4>;
    } else {
        ws->nw = 8;
        ws->ns = 4;
        ws->fn = (const void*)k_wstep<1, 8, 4>;
    }
    const int WK = 4 * w + 42 * m;
    ws->smem = ws->nw * ws->ns * ws->BS * 4 + ws->nw * ws->ns * 8 + ws->nw * WK * 4;
    SFW_CUDA_TRY(cudaFuncSetAttribute(ws->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ws->smem));
    g_wf[h] = ws;
    return 0;
}

// Convert U-form vectors (sources, probe weights, states) to W-form and upload
// sources/probes in fp32.  src_vec/probe_w: HOST U-form arrays as given at create/set_probes.
extern "C" int sfw_wform_vectors(sfw_stepper* h, const double* src_vec, const double* probe_w, double* src_norms,
                                 char* errbuf, int errlen) {
    WState* ws = g_wf.count(h) ? g_wf[h] : nullptr;
    if (!ws) return fail(SFW_ECONFIG, "call sfw_wform_setup first", errbuf, errlen);
    int rc = 0;
    // sources: w = G^-1 src  (U = G W)
    if (h->n_src) {
        std::vector<int> vs(h->n_src);
        std::vector<long long> vo(h->n_src);
        long long tot = 0;
        std::vector<int> sp(h->n_sub + 1);
        cudaMemcpy(sp.data(), h->src_ptr, (h->n_sub + 1) * 4, cudaMemcpyDeviceToHost);
        std::vector<int> sid(h->n_src);
        cudaMemcpy(sid.data(), h->src_ids, h->n_src * 4, cudaMemcpyDeviceToHost);
        for (int s = 0; s < h->n_sub; ++s)
            for (int q = sp[s]; q < sp[s + 1]; ++q) vs[sid[q]] = s;
        for (int i = 0; i < h->n_src; ++i) {
            vo[i] = tot;
            tot += h->soff[vs[i] + 1] - h->soff[vs[i]];
        }
        std::vector<double> out(tot);
        if ((rc = wf_vectors(h, ws, h->n_src, vs.data(), vo.data(), tot, 0, src_vec, out.data(), errbuf, errlen)))
            return rc;
        if (src_norms)
            for (int i = 0; i < h->n_src; ++i) {
                const long long len = h->soff[vs[i] + 1] - h->soff[vs[i]];
                double t = 0.0;
                for (long long e = 0; e < len; ++e) t += out[vo[i] + e] * out[vo[i] + e];
                src_norms[i] = std::sqrt(t);
            }
        std::vector<float> f(out.begin(), out.end());
        if (ws->src) cudaFree(ws->src);
        ws->src = nullptr;
        if ((rc = upload(&ws->src, f, errbuf, errlen))) return rc;
    }
    // probes: weights^W = G^T weights^U
    if (h->n_probe) {
        std::vector<int> pp(h->n_sub + 1), pid(h->n_probe);
        cudaMemcpy(pp.data(), h->prb_ptr, (h->n_sub + 1) * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(pid.data(), h->prb_ids, h->n_probe * 4, cudaMemcpyDeviceToHost);
        std::vector<int> vs(h->n_probe);
        std::vector<long long> vo(h->n_probe);
        for (int s = 0; s < h->n_sub; ++s)
            for (int q = pp[s]; q < pp[s + 1]; ++q) vs[pid[q]] = s;
        long long tot = 0;
        for (int i = 0; i < h->n_probe; ++i) {
            vo[i] = tot;
            tot += h->soff[vs[i] + 1] - h->soff[vs[i]];
        }
        std::vector<double> out(tot);
        if ((rc = wf_vectors(h, ws, h->n_probe, vs.data(), vo.data(), tot, 1, probe_w, out.data(), errbuf, errlen)))
            return rc;
        std::vector<float> f(out.begin(), out.end());
        if (ws->prb) cudaFree(ws->prb);
        ws->prb = nullptr;
        if ((rc = upload(&ws->prb, f, errbuf, errlen))) return rc;
    }
    return 0;
}

static int wf_launch(sfw_stepper* h, WState* ws, int mode, int n_steps, int record_every, int ftab_stride, char* errbuf,
                     int errlen) {
    WParams p{};
    p.n_sub = h->n_sub;
    p.L = h->L;
    p.BS = ws->BS;
    p.n_steps = n_steps;
    p.record_every = record_every;
    p.n_probe = h->n_probe;
    p.ftab_stride = ftab_stride;
    p.mode = mode;
    p.dt = h->dt;
    p.dt2 = (float)(h->dt * h->dt);
    p.half = (float)((0.5 * h->dt) * h->dt);
    p.coef = ws->coef;
    p.W0 = ws->W[ws->cur];
    p.W1 = ws->W[ws->cur ^ 1];
    p.V0 = ws->V0;
    p.P = ws->P;
    p.Cc = ws->Cc;
    p.cta_sub_ptr = h->cta_sub_ptr;
    p.nbr = h->nbr;
    p.src_ptr = h->src_ptr;
    p.src_ids = h->src_ids;
    p.src_vec = ws->src;
    p.src_voff = h->src_voff;
    p.ftab = ws->ftab;
    p.prb_ptr = h->prb_ptr;
    p.prb_ids = h->prb_ids;
    p.prb_tap = h->prb_tap;
    p.prb_w = ws->prb;
    p.prb_woff = h->prb_woff;
    p.rows = h->rows;
    p.sub_norm = h->sub_norm;
    p.sqs = ws->sqs;
    p.norm_part = h->norm_part;
    p.flags = h->bar;
    p.ncta_ptr = h->ncta_ptr;
    p.ncta = h->ncta;
    SFW_CUDA_TRY(cudaMemsetAsync(h->bar, 0, sizeof(unsigned int) * h->grid, h->stream));
    void* args[] = {&p};
    SFW_CUDA_TRY(cudaLaunchCooperativeKernel(ws->fn, dim3(h->grid), dim3(ws->nw * 32), args, ws->smem, h->stream));
    return 0;
}

static int wf_ensure(float** p, long long* cap, long long need, char* errbuf, int errlen) {
    if (*cap >= need && *p) return 0;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    int rc = dalloc(p, need, errbuf, errlen);
    if (!rc) *cap = need;
    return rc;
}

// Two-level start in W-form.  u0/v0: HOST U-form (or NULL); converted with G^-1.
extern "C" int sfw_wform_init(sfw_stepper* h, const double* u0, const double* v0, const double* profile0,
                              double* row0_out, char* errbuf, int errlen) {
    WState* ws = g_wf.count(h) ? g_wf[h] : nullptr;
    if (!ws) return fail(SFW_ECONFIG, "call sfw_wform_setup first", errbuf, errlen);
    const long long n = h->state_len;
    ws->cur = 0;
    std::vector<int> vs(h->n_sub);
    std::vector<long long> vo(h->n_sub);
    for (int s = 0; s < h->n_sub; ++s) {
        vs[s] = s;
        vo[s] = h->soff[s];
    }
    int rc = 0;
    for (int which = 0; which < 2; ++which) {
        const double* src = which == 0 ? u0 : v0;
        float* dst = nullptr;
        if (which == 0) {
            dst = ws->W[0];
        } else {
            if (!src) {
                if (ws->V0) cudaMemset(ws->V0, 0, n * 4);
                continue;
            }
            if (!ws->V0 && (rc = dalloc(&ws->V0, n, errbuf, errlen))) return rc;
            dst = ws->V0;
        }
        if (!src) {
            cudaMemset(dst, 0, n * 4);
            continue;
        }
        std::vector<double> out(n);
        if ((rc = wf_vectors(h, ws, h->n_sub, vs.data(), vo.data(), n, 0, src, out.data(), errbuf, errlen))) return rc;
        std::vector<float> f(out.begin(), out.end());
        cudaMemcpy(dst, f.data(), n * 4, cudaMemcpyHostToDevice);
    }
    if ((rc = wf_ensure(&ws->ftab, &ws->ftab_cap, std::max(1, h->n_src), errbuf, errlen))) return rc;
    if (h->n_src) {
        std::vector<float> f(profile0, profile0 + h->n_src);
        cudaMemcpy(ws->ftab, f.data(), h->n_src * 4, cudaMemcpyHostToDevice);
    }
    // row buffer / norm partials owned by the fp64 handle
    double* tmp = nullptr;
    (void)tmp;
    if (!h->rows || h->rows_cap < std::max(1, h->n_probe)) {
        if (h->rows) cudaFree(h->rows);
        h->rows = nullptr;
        if ((rc = dalloc(&h->rows, std::max(1, h->n_probe), errbuf, errlen))) return rc;
        h->rows_cap = std::max(1, h->n_probe);
    }
    if (!h->norm_part || h->norm_cap < h->grid) {
        if (h->norm_part) cudaFree(h->norm_part);
        h->norm_part = nullptr;
        if ((rc = dalloc(&h->norm_part, h->grid, errbuf, errlen))) return rc;
        h->norm_cap = h->grid;
    }
    if ((rc = wf_launch(h, ws, 1, 1, 1, 1, errbuf, errlen))) return rc;
    if (row0_out && h->n_probe)
        SFW_CUDA_TRY(cudaMemcpyAsync(row0_out, h->rows, h->n_probe * 8, cudaMemcpyDeviceToHost, h->stream));
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    return 0;
}

// n_steps fp32 W-form leapfrog steps (one launch).  Same table conventions as sfw_step_run;
// norms are |W| (the W-form invariant scale), rows are the physical probe values.
extern "C" int sfw_wform_run(sfw_stepper* h, int n_steps, int record_every, const double* profile,
                             double* rows_out, double* norms_out, float* kernel_ms, char* errbuf, int errlen) {
    WState* ws = g_wf.count(h) ? g_wf[h] : nullptr;
    if (!ws) return fail(SFW_ECONFIG, "call sfw_wform_setup first", errbuf, errlen);
    if (n_steps <= 0) return 0;
    int rc = wf_ensure(&ws->ftab, &ws->ftab_cap, std::max(1LL, (long long)h->n_src * n_steps), errbuf, errlen);
    if (rc) return rc;
    if (h->n_src && profile) {
        std::vector<float> f(profile, profile + (size_t)h->n_src * n_steps);
        cudaMemcpy(ws->ftab, f.data(), f.size() * 4, cudaMemcpyHostToDevice);
    }
    const long long nrec = n_steps / record_every;
    if (h->rows_cap < std::max(1LL, nrec * h->n_probe)) {
        if (h->rows) cudaFree(h->rows);
        h->rows = nullptr;
        if ((rc = dalloc(&h->rows, std::max(1LL, nrec * h->n_probe), errbuf, errlen))) return rc;
        h->rows_cap = std::max(1LL, nrec * h->n_probe);
    }
    if (h->norm_cap < (long long)n_steps * h->grid) {
        if (h->norm_part) cudaFree(h->norm_part);
        h->norm_part = nullptr;
        if ((rc = dalloc(&h->norm_part, (size_t)n_steps * h->grid, errbuf, errlen))) return rc;
        h->norm_cap = (long long)n_steps * h->grid;
    }
    SFW_CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
    if ((rc = wf_launch(h, ws, 0, n_steps, record_every, n_steps, errbuf, errlen))) return rc;
    SFW_CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
    ws->cur ^= (n_steps & 1);
    std::vector<double> part((size_t)n_steps * h->grid);
    if (rows_out && nrec * h->n_probe > 0)
        SFW_CUDA_TRY(cudaMemcpyAsync(rows_out, h->rows, (size_t)nrec * h->n_probe * 8, cudaMemcpyDeviceToHost, h->stream));
    if (norms_out)
        SFW_CUDA_TRY(cudaMemcpyAsync(part.data(), h->norm_part, part.size() * 8, cudaMemcpyDeviceToHost, h->stream));
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    if (kernel_ms) cudaEventElapsedTime(kernel_ms, h->ev0, h->ev1);
    if (norms_out)
        for (int k = 0; k < n_steps; ++k) {
            double t = 0.0;
            for (int c = 0; c < h->grid; ++c) t += part[(size_t)k * h->grid + c];
            norms_out[k] = std::sqrt(t);
        }
    return 0;
}

// W-form state as U-form (U_j = G_j W_j), fp64, HOST concat.
extern "C" int sfw_wform_state(sfw_stepper* h, double* u_curr, double* u_prev, char* errbuf, int errlen) {
    WState* ws = g_wf.count(h) ? g_wf[h] : nullptr;
    if (!ws) return fail(SFW_ECONFIG, "call sfw_wform_setup first", errbuf, errlen);
    const long long n = h->state_len;
    std::vector<int> vs(h->n_sub);
    std::vector<long long> vo(h->n_sub);
    for (int s = 0; s < h->n_sub; ++s) {
        vs[s] = s;
        vo[s] = h->soff[s];
    }
    for (int lvl = 0; lvl < 2; ++lvl) {
        double* dst = lvl == 0 ? u_curr : u_prev;
        if (!dst) continue;
        std::vector<float> f(n);
        cudaMemcpy(f.data(), ws->W[lvl == 0 ? ws->cur : ws->cur ^ 1], n * 4, cudaMemcpyDeviceToHost);
        std::vector<double> in(f.begin(), f.end());
        int rc = wf_vectors(h, ws, h->n_sub, vs.data(), vo.data(), n, 2, in.data(), dst, errbuf, errlen);
        if (rc) return rc;
    }
    return 0;
}

// bytes per step of the fp32 W-form launch (4[(2L-1)w(w+1)/2 + 3Lw] per subdomain)
extern "C" int sfw_wform_traffic(sfw_stepper* h, double* alg_bytes, double* streamed) {
    const double w = h->W;
    double b = 0, s = 0;
    const int BS = wf::packed_stride32(h->m);
    for (int i = 0; i < h->n_sub; ++i) {
        const double L = h->layers[i];
        b += 4.0 * ((2 * L - 1) * w * (w + 1) / 2 + 3 * L * w);
        s += 4.0 * ((2 * L - 1) * BS + 3 * L * w);
    }
    if (alg_bytes) *alg_bytes = b;
    if (streamed) *streamed = s;
    return 0;
}

extern "C" int sfw_wform_destroy(sfw_stepper* h) {
    if (!g_wf.count(h)) return 0;
    WState* ws = g_wf[h];
    void* ptrs[] = {ws->coef, ws->W[0], ws->W[1], ws->V0, ws->P, ws->Cc, ws->src, ws->prb, ws->ftab, ws->sqs,
                    ws->first_blk};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    delete ws;
    g_wf.erase(h);
    return 0;
}
