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

// Packed fp32 block (symmetric A_j, or lower-triangular B_j^T), laid out for 16-B shared loads.
// A w x w block (w = 6m) is 15 off-diagonal m x m tiles t = (I > K) plus 6 diagonal lower
// triangles d.  Inside a tile, element e <-> (r, c) = (e % m, (e / m + e % m) % m) (wrapped
// diagonals: m consecutive e touch m distinct rows and columns).  Inside a triangle, element
// q = dd*m - dd(dd-1)/2 + c holds row c + dd, column c.  Storage (floats):
//   [tile chunks]  (e/4)*60 + t*4 + e%4             for e < 4*NC,  NC  = m*m/4
//   [tri chunks]   60*NC + (q/4)*24 + d*4 + q%4     for q < 4*NC2, NC2 = tri/4
//   [tile tails]   60*NC + 24*NC2 + (e-4NC)*15 + t
//   [tri tails]    60*NC + 24*NC2 + 15*(m*m%4) + (q-4NC2)*6 + d
// so the 15 tile lanes (or 6 triangle lanes) of a warp read one float4 each per LDS.128.
__host__ __device__ constexpr int nc1(int m) { return (m * m) / 4; }
__host__ __device__ constexpr int nc2(int m) { return tri_count(m) / 4; }
__host__ __device__ constexpr int tri_base(int m) { return 60 * nc1(m); }
__host__ __device__ constexpr int tail1_base(int m) { return 60 * nc1(m) + 24 * nc2(m); }
__host__ __device__ constexpr int tail2_base(int m) { return tail1_base(m) + 15 * ((m * m) % 4); }
__host__ __device__ inline int off_pos(int m, int t, int e) {
    return e < 4 * nc1(m) ? (e / 4) * 60 + t * 4 + (e % 4) : tail1_base(m) + (e - 4 * nc1(m)) * 15 + t;
}
__host__ __device__ inline int diag_pos(int m, int d, int q) {
    return q < 4 * nc2(m) ? tri_base(m) + (q / 4) * 24 + d * 4 + (q % 4) : tail2_base(m) + (q - 4 * nc2(m)) * 6 + d;
}
__host__ __device__ constexpr int tri_row0(int m, int dd) { return dd * m - dd * (dd - 1) / 2; }
__host__ __device__ constexpr int tri_dd(int m, int q) {
    int dd = 0;
    while (q >= tri_row0(m, dd + 1)) ++dd;
    return dd;
}
__host__ __device__ inline int packed_pos(int m, int row, int col) {
    const int I = row / m, K = col / m, r = row % m, c = col % m;
    if (I != K) return off_pos(m, off_tile(I, K), ((c - r + m) % m) * m + r);
    const int dd = r - c;
    return diag_pos(m, I, dd * m - dd * (dd - 1) / 2 + c);
}
}  // namespace wf

// Partial-sum slots of the paired block product (per output row r of a tile group, stride PS):
//   [0,15)  tile t rows I: A_j + B_j^T row partials      -> p_j
//   [15,30) tile t rows K: A_j column partials            -> p_j
//   [30,45) tile t rows K: B_j column partials (B_j W_j)  -> c_{j+1}
//   [45,51) triangle d:    A_j (both parts) + B_j^T rows  -> p_j
//   [51,57) triangle d:    B_j column partials            -> c_{j+1}
//   57      zero
constexpr int PS = 61;  // 57 zero slot, 58-60 junk slots of idle lanes

template <int M>
struct WRed2 {
    static constexpr int W = 6 * M, EPL = (W + 31) / 32;
    int po[EPL][6], co[EPL][6];
    __device__ __forceinline__ explicit WRed2(int lane) {
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            const int i = lane + 32 * e;
            const int R = i < W ? i / M : 0, r = i < W ? i % M : 0;
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                // p_j: tiles (R, K < R) rows, tiles (I > R, R) columns, triangle R
                po[e][q] = q < R ? r * PS + wf::off_tile(R, q)
                                 : q < 5 ? r * PS + 15 + wf::off_tile(q + 1, R) : r * PS + 45 + R;
                // c_{j+1}: tiles (I > R, R) columns of B_j, triangle R, zero slot
                co[e][q] = q < 5 - R ? r * PS + 30 + wf::off_tile(R + 1 + q, R)
                                     : q == 5 - R ? r * PS + 51 + R : r * PS + 57;
            }
        }
    }
};

// One warp, one pass over the pair (A_j, B_j^T) staged in shared memory:
//   half 0 (lanes 0-15) reads A_j, half 1 (lanes 16-31) reads B_j^T.
//   p_j = A_j x_j + B_j^T x_{j+1},   c_{j+1} = B_j x_j     (partials into `part`, summed by WRed2)
// Control flow is warp-uniform: idle lanes (t = 15 in the tile pass, t >= 6 in the triangle
// pass, half 1 when !hasB) run the same code on finite shared data with x = 0 and store to
// junk slots, so the warp never splits (a split warp runs each half separately).
template <int M>
__device__ __forceinline__ void wpair(const float* __restrict__ blkA, const float* xj, const float* xj1, float* part,
                                      int lane, bool hasB, int BS) {
    constexpr int MM = M * M, NC = wf::nc1(M), TRI = wf::tri_count(M), NC2 = wf::nc2(M);
    const int h = lane >> 4, t = lane & 15;
    const float* blk = blkA + h * BS;
    const bool act = (h == 0) || hasB;
    const float* xv = h ? xj1 : xj;
    {
        const int tt = t < 15 ? t : 14;
        const float xs = (t < 15 && act) ? 1.f : 0.f;
        const int I = wf::off_I(tt), K = wf::off_K(tt);
        float P[M], Q[M], xk[M], xi[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            xk[i] = xv[K * M + i] * xs;
            xi[i] = xj[I * M + i] * xs;
            P[i] = Q[i] = 0.f;
        }
#pragma unroll
        for (int ch = 0; ch < NC; ++ch) {
            const float4 a4 = *reinterpret_cast<const float4*>(blk + ch * 60 + tt * 4);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = ch * 4 + u, r = e % M, c = (e / M + r) % M;
                P[r] = fmaf(av[u], xk[c], P[r]);
                Q[c] = fmaf(av[u], xi[r], Q[c]);
            }
        }
#pragma unroll
        for (int e = 4 * NC; e < MM; ++e) {
            const int r = e % M, c = (e / M + r) % M;
            const float a = blk[wf::tail1_base(M) + (e - 4 * NC) * 15 + tt];
            P[r] = fmaf(a, xk[c], P[r]);
            Q[c] = fmaf(a, xi[r], Q[c]);
        }
        const int sa = t == 15 ? 58 : (h ? 30 + t : t);  // h0: A+B^T rows I; h1: B columns K
        const int sb = (t == 15 || h) ? 59 : 15 + t;       // h0: A columns K
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const float ps = P[i] + __shfl_xor_sync(0xffffffffu, P[i], 16);
            part[i * PS + sa] = h ? Q[i] : ps;
            part[i * PS + sb] = Q[i];
        }
    }
    {
        const int d = t < 6 ? t : 5;
        const float xs = (t < 6 && act) ? 1.f : 0.f;
        const float qsel = h ? 1.f : 0.f;  // symmetric block: diagonal counted once
        float P[M], Q[M], xa[M], xb[M];
#pragma unroll
        for (int i = 0; i < M; ++i) {
            xa[i] = xv[d * M + i] * xs;
            xb[i] = xj[d * M + i] * xs;
            P[i] = Q[i] = 0.f;
        }
        auto term = [&](int q, float a) {
            const int dd = wf::tri_dd(M, q), c = q - wf::tri_row0(M, dd), r = c + dd;
            P[r] = fmaf(a, xa[c], P[r]);
            Q[c] = fmaf(dd == 0 ? a * qsel : a, xb[r], Q[c]);
        };
#pragma unroll
        for (int ch = 0; ch < NC2; ++ch) {
            const float4 a4 = *reinterpret_cast<const float4*>(blk + wf::tri_base(M) + ch * 24 + d * 4);
            term(ch * 4 + 0, a4.x);
            term(ch * 4 + 1, a4.y);
            term(ch * 4 + 2, a4.z);
            term(ch * 4 + 3, a4.w);
        }
#pragma unroll
        for (int q = 4 * NC2; q < TRI; ++q) term(q, blk[wf::tail2_base(M) + (q - 4 * NC2) * 6 + d]);
        const int sa = t >= 6 ? 60 : (h ? 51 + t : 45 + t);
#pragma unroll
        for (int i = 0; i < M; ++i) {
            float D = h ? P[i] : P[i] + Q[i];
            D += __shfl_xor_sync(0xffffffffu, D, 16);
            part[i * PS + sa] = h ? Q[i] : D;
        }
    }
}

struct WParams {
    int n_sub, L, BS, n_steps, record_every, n_probe, ftab_stride, mode;  // mode 0 step, 1 init
    unsigned int tag0;      // mailbox tag of step k is tag0 + k (monotone across launches)
    double dt;
    float dt2, half;
    const float* coef;      // [n_sub][2L-1][BS]: A_0, B_0^T, A_1, B_1^T, ..., A_{L-1}
    float* W0;              // current level (read)
    float* W1;              // previous level, overwritten with the next level
    const float* V0;        // init velocity (W-form) or null
    unsigned long long* mbox;  // [2][n_sub][W] tagged layer-0 partials p_0 (face mailbox)
    const int* cta_sub_ptr;
    const int* nbr;
    const int* src_ptr;
    const int* src_ids;
    const float* src_vec;   // W-form source vectors
    const long long* src_voff;
    const float* ftab;      // [n_src][ftab_stride] profile values
    const int* prb_ptr;
    const int* prb_ids;
    const float* prb_w;     // W-form probe weights
    const long long* prb_woff;
    const int* prb_rng;     // [n_probe][2]: first element, element count of the nonzero layer range
    double* rows;
    double* norm_part;      // [n_steps][grid * NW]
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

__device__ __forceinline__ void st_tagged(unsigned long long* p, float v, unsigned int tag) {
    const unsigned long long w = ((unsigned long long)tag << 32) | (unsigned long long)__float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

// warp-uniform mbarrier wait: every lane polls, the warp leaves the loop together
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
    while (!__all_sync(0xffffffffu, mbar_try_wait(bar, parity))) {
    }
}

// fp32 W-form stepping, persistent (one launch = n_steps steps).  Warp-per-subdomain:
// each warp owns subdomains s0+warp, s0+warp+NW, ... and sweeps their layers in order,
// so the carry c_j = B_{j-1} W_{j-1} stays in registers and the leapfrog of layers j >= 1
// is fused into the block pass.  Layer 0 waits for the neighbours' p_0 face slices,
// which travel through a tagged mailbox (value and step tag in one 64-bit word): no
// CTA barrier, no flag round trip.  The (A_j, B_j^T) pair of each item is one TMA bulk
// copy into a per-warp NS-deep ring.  All control flow inside the step loop is
// warp-uniform (lane-dependent work is predicated), so the warp never splits.
template <int M, int NS>
__global__ void __launch_bounds__(256, 1) k_wstep(const WParams p) {
    constexpr int W = 6 * M;
    constexpr int EPL = (W + 31) / 32;
    const int NW = blockDim.x >> 5;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const WRed2<M> ro(lane);
    const int BS = p.BS, L = p.L;
    const long long K = (long long)L * W;
    const int PAIR = 2 * BS;
    float* stages = reinterpret_cast<float*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + (size_t)NW * NS * PAIR);
    float* wk = reinterpret_cast<float*>(bars + NW * NS) + (size_t)warp * (2 * W + M * PS);
    float* buf = wk;           // [2][W]: W_j, W_{j+1} of the current item (ring by layer parity)
    float* part = wk + 2 * W;  // [M][PS]
    float* my_stage = stages + (size_t)warp * NS * PAIR;
    uint64_t* my_bar = bars + warp * NS;
    // stage memory must hold finite values (idle lanes multiply stale data by 0)
    for (int i = lane; i < NS * PAIR; i += 32) my_stage[i] = 0.f;
    for (int i = lane; i < M * PS; i += 32) part[i] = 0.f;
    for (int i = lane; i < 2 * W; i += 32) buf[i] = 0.f;
    if (lane == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&my_bar[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int s0 = p.cta_sub_ptr[blockIdx.x], s1 = p.cta_sub_ptr[blockIdx.x + 1];
    const int n_my = (s1 - s0) > warp ? (s1 - s0 - warp + NW - 1) / NW : 0;
    const int n_iter = p.mode == 0 ? p.n_steps : 1;
    const long long total = (long long)n_my * L * n_iter;
    const uint64_t pol = l2_policy_evict_first();
    long long issued = 0, consumed = 0;
    int pr_t = 0, pr_j = 0;
    auto issue = [&]() {  // warp-uniform bookkeeping, lane 0 issues
        while (issued < total && issued < consumed + NS) {
            const int s = s0 + warp + pr_t * NW;
            const long long blk = (long long)s * (2 * L - 1) + 2 * pr_j;
            const uint32_t bytes = (uint32_t)((pr_j + 1 < L ? 2 : 1) * BS) * 4u;
            const int st = (int)(issued % NS);
            if (lane == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(&my_bar[st], bytes);
                bulk_g2s(my_stage + (size_t)st * PAIR, p.coef + blk * BS, bytes, &my_bar[st], pol);
            }
            ++issued;
            if (++pr_j == L) {
                pr_j = 0;
                if (++pr_t == n_my) pr_t = 0;
            }
        }
    };
    issue();
    const float dt = (float)p.dt, dt2 = p.dt2, half = p.half;
    const int NWG = gridDim.x * NW;
    bool ok_e[EPL];
    int ic[EPL];  // this lane's rows (clamped; stores predicated on ok_e)
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        ok_e[e] = lane + 32 * e < W;
        ic[e] = ok_e[e] ? lane + 32 * e : W - 1;
    }

    for (int k = 1; k <= n_iter; ++k) {
        const unsigned int tag = p.tag0 + (unsigned int)k;
        unsigned long long* mb = p.mbox + (size_t)(tag & 1u) * p.n_sub * W;
        const int cb = (k - 1) & 1;  // W0 holds the current level at k = 1
        const float* Wc = cb ? p.W1 : p.W0;
        float* Wn = cb ? p.W0 : p.W1;
        const int kk = k - 1;
        double sq = 0.0;  // this lane's share of |W_next|^2 (fixed order)
        // ---------------- layers 1..L-1 (fused), layer-0 partials to the mailbox ------------
        float na[EPL], nb[EPL];  // prefetch for the next item
        auto prefetch = [&](int t, int j) {
            const int s = s0 + warp + t * NW;
            const float* w = Wc + (size_t)s * K;
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                const int i = ic[e];
                if (j == 0) {
                    na[e] = w[i];
                    nb[e] = L > 1 ? w[W + i] : 0.f;
                } else {
                    na[e] = j + 1 < L ? w[(size_t)(j + 1) * W + i] : 0.f;
                    nb[e] = p.mode == 0 ? Wn[(size_t)s * K + (size_t)j * W + i] : 0.f;
                }
            }
        };
        if (n_my > 0) prefetch(0, 0);
        float carry[EPL], wprev[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) carry[e] = wprev[e] = 0.f;
        for (int t = 0; t < n_my; ++t) {
            const int s = s0 + warp + t * NW;
            const bool has_src = p.src_ptr[s] != p.src_ptr[s + 1];
            for (int j = 0; j < L; ++j) {
                float* xj = buf + (j & 1) * W;
                float* xj1 = buf + ((j + 1) & 1) * W;
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    if (j == 0) {
                        if (ok_e[e]) {
                            xj[ic[e]] = na[e];
                            xj1[ic[e]] = nb[e];
                        }
                        carry[e] = 0.f;
                    } else {
                        if (ok_e[e]) xj1[ic[e]] = na[e];
                        wprev[e] = nb[e];
                    }
                }
                __syncwarp();
                if (j + 1 < L)
                    prefetch(t, j + 1);
                else if (t + 1 < n_my)
                    prefetch(t + 1, 0);
                const int st = (int)(consumed % NS);
                mbar_wait_warp(&my_bar[st], (uint32_t)((consumed / NS) & 1));
                wpair<M>(my_stage + (size_t)st * PAIR, xj, xj1, part, lane, j + 1 < L, BS);
                __syncwarp();
                ++consumed;
                issue();
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    float pj = part[ro.po[e][0]];
#pragma unroll
                    for (int q = 1; q < 6; ++q) pj += part[ro.po[e][q]];
                    float cn = part[ro.co[e][0]];
#pragma unroll
                    for (int q = 1; q < 6; ++q) cn += part[ro.co[e][q]];
                    if (j == 0) {
                        if (ok_e[e]) st_tagged(mb + (size_t)s * W + ic[e], pj, tag);
                    } else {
                        const size_t o = (size_t)s * K + (size_t)j * W + ic[e];
                        float tot = pj + carry[e];
                        if (has_src) tot = wforce(p, s, (long long)j * W + ic[e], kk, tot);
                        const float v = (p.mode == 1 && p.V0) ? p.V0[o] : 0.f;
                        const float un = wleap(p.mode, xj[ic[e]], wprev[e], v, tot, dt, dt2, half);
                        if (ok_e[e]) {
                            Wn[o] = un;
                            sq = fma((double)un, (double)un, sq);
                        }
                    }
                    carry[e] = cn;
                }
                __syncwarp();
            }
        }
        // ---------------- layer 0: faces (mailbox), leapfrog -------------------------------
        for (int t = 0; t < n_my; ++t) {
            const int s = s0 + warp + t * NW;
            const size_t o = (size_t)s * K;
            const bool has_src = p.src_ptr[s] != p.src_ptr[s + 1];
            const unsigned long long* own[EPL];
            const unsigned long long* nbp[EPL];
            float wc[EPL], wo[EPL], v[EPL];
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                const int i = ic[e], f = i / M;
                const int nbs = p.nbr[s * 6 + f];
                own[e] = mb + (size_t)s * W + i;
                nbp[e] = nbs >= 0 ? mb + (size_t)nbs * W + (f ^ 1) * M + i % M : own[e];
                wc[e] = Wc[o + i];
                wo[e] = (p.mode == 0) ? Wn[o + i] : 0.f;
                v[e] = (p.mode == 1 && p.V0) ? p.V0[o + i] : 0.f;
            }
            float a[EPL], b[EPL];
            int spins = 0;
            while (true) {  // warp-uniform poll of the tagged face words
                bool ok = true;
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    const unsigned long long wa = ld_relaxed64(own[e]);
                    const unsigned long long wb = ld_relaxed64(nbp[e]);
                    ok = ok && (unsigned int)(wa >> 32) == tag && (unsigned int)(wb >> 32) == tag;
                    a[e] = __uint_as_float((unsigned int)wa);
                    b[e] = __uint_as_float((unsigned int)wb);
                }
                if (__all_sync(0xffffffffu, ok)) break;
                if (++spins > 2) __nanosleep(100);
            }
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                const int i = ic[e];
                float tot = (nbp[e] != own[e]) ? 0.5f * (a[e] + b[e]) : a[e];
                if (has_src) tot = wforce(p, s, i, kk, tot);
                const float un = wleap(p.mode, wc[e], wo[e], v[e], tot, dt, dt2, half);
                if (ok_e[e]) {
                    Wn[o + i] = un;
                    sq = fma((double)un, (double)un, sq);
                }
            }
        }
        __syncwarp();
        if (p.mode == 0) {
            const double vs = warp_sum(sq);
            if (lane == 0) p.norm_part[(size_t)kk * NWG + blockIdx.x * NW + warp] = vs;
        }
        // probes: all layers of this warp's subdomains are written
        const bool rec = (p.mode == 1) || (k % p.record_every == 0);
        if (rec && p.rows) {
            const long long row = (p.mode == 1) ? 0 : (k / p.record_every - 1);
            for (int t = 0; t < n_my; ++t) {
                const int s = s0 + warp + t * NW;
                const float* U = ((p.mode == 1) ? Wc : Wn) + (size_t)s * K;
                const int pa = p.prb_ptr[s], pb = p.prb_ptr[s + 1];
                // short probes (receiver-face coefficients, <= 64 weights): one per lane, 32 at a
                // time, a sequential sum; long ones (node receivers over the whole state) warp-
                // cooperatively.  The path depends on the probe's own length only, so a probe's value
                // does not depend on which other probes share its subdomain.
                for (int q0 = pa; q0 < pb; q0 += 32) {
                    const int q = q0 + lane;
                    if (q < pb) {
                        const int pid = p.prb_ids[q];
                        const int lo = p.prb_rng[2 * pid], cnt = p.prb_rng[2 * pid + 1];
                        if (cnt <= 64) {
                            const float* wv = p.prb_w + p.prb_woff[pid];
                            double val = 0.0;
                            for (int i = lo; i < lo + cnt; ++i) val = fma((double)wv[i], (double)U[i], val);
                            p.rows[row * p.n_probe + pid] = val;
                        }
                    }
                }
                for (int pq = pa; pq < pb; ++pq) {
                    if (p.prb_rng[2 * p.prb_ids[pq] + 1] <= 64) continue;
                    const int pid = p.prb_ids[pq];
                    const int lo = p.prb_rng[2 * pid], cnt = p.prb_rng[2 * pid + 1];
                    const float* wv = p.prb_w + p.prb_woff[pid];
                    double val = 0.0;
                    for (int b0 = 0; b0 < cnt; b0 += 32) {
                        const int i = lo + b0 + lane;
                        if (b0 + lane < cnt) val = fma((double)wv[i], (double)U[i], val);
                    }
                    val = warp_sum(val);
                    if (lane == 0) p.rows[row * p.n_probe + pid] = val;
                }
            }
        }
        __syncwarp();
    }
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
    float *coef = nullptr, *W[2] = {nullptr, nullptr}, *V0 = nullptr;
    float *src = nullptr, *prb = nullptr, *ftab = nullptr;
    long long ftab_cap = 0;
    unsigned long long* mbox = nullptr;  // [2][n_sub][w] tagged layer-0 partials
    unsigned int tag = 0;                // last mailbox tag used
    int* prb_rng = nullptr;              // [n_probe][2]
    double* norm = nullptr;              // [n_steps][grid * nw] per-warp |W|^2 partials
    long long norm_cap = 0;
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
    sfw_h2d(d_in, in_host, n * 8);
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
    struct WScope { WScope() { ++sfw::g_wform_scope; } ~WScope() { --sfw::g_wform_scope; } } wscope_;
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
        (rc = dalloc(&ws->mbox, (size_t)2 * n * w, errbuf, errlen)))
        return rc;
    cudaMemsetAsync(ws->coef, 0, (size_t)nb * ws->BS * 4, h->stream);
    cudaMemsetAsync(ws->mbox, 0, (size_t)2 * n * w * 8, h->stream);
    const size_t sm = (size_t)3 * w * w * 8;
    SFW_CUDA_TRY(cudaFuncSetAttribute(k_wform_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_wform_blocks<<<(unsigned)ls.size(), 256, sm, h->stream>>>(h->scales, h->gam_dense, d_ls, d_lj, ws->first_blk,
                                                                h->d_layers, m, ws->BS, ws->coef);
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    cudaFree(d_ls);
    cudaFree(d_lj);
    // launch shape: one CTA per SM (h->grid), NW warps, each owning whole subdomains.
    // NW = ceil(spc / rounds) with rounds = ceil(spc / 8) balances the per-warp subdomain count.
    int spc = 1;
    for (int b = 0; b < h->grid; ++b) spc = std::max(spc, h->cta_ptr_h[b + 1] - h->cta_ptr_h[b]);
    const int rounds = (spc + 7) / 8;
    ws->nw = std::max(1, std::min(8, (spc + rounds - 1) / rounds));
    if (const char* e = getenv("SFW_WSTEP_NW")) ws->nw = std::max(1, std::min(8, atoi(e)));  // test hook
    ws->ns = 2;
    if (m == 9)
        ws->fn = (const void*)k_wstep<9, 2>;
    else if (m == 4)
        ws->fn = (const void*)k_wstep<4, 2>;
    else
        ws->fn = (const void*)k_wstep<1, 2>;
    ws->smem = ws->nw * (ws->ns * 2 * ws->BS * 4 + ws->ns * 8 + (2 * w + m * PS) * 4);
    SFW_CUDA_TRY(cudaFuncSetAttribute(ws->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ws->smem));
    g_wf[h] = ws;
    return 0;
}

// Convert U-form vectors (sources, probe weights, states) to W-form and upload
// sources/probes in fp32.  src_vec/probe_w: HOST U-form arrays as given at create/set_probes.
extern "C" int sfw_wform_vectors(sfw_stepper* h, const double* src_vec, const double* probe_w, double* src_norms,
                                 char* errbuf, int errlen) {
    struct WScope { WScope() { ++sfw::g_wform_scope; } ~WScope() { --sfw::g_wform_scope; } } wscope_;
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
        // nonzero element range of each W-form probe (face-coefficient probes live in layer 0)
        std::vector<int> rng(2 * h->n_probe, 0);
        for (int i = 0; i < h->n_probe; ++i) {
            const long long len = h->soff[vs[i] + 1] - h->soff[vs[i]];
            long long lo = 0, hi = len;
            while (lo < len && f[vo[i] + lo] == 0.f) ++lo;
            while (hi > lo && f[vo[i] + hi - 1] == 0.f) --hi;
            rng[2 * i] = (int)lo;
            rng[2 * i + 1] = (int)(hi - lo);
        }
        if (ws->prb_rng) cudaFree(ws->prb_rng);
        ws->prb_rng = nullptr;
        if ((rc = upload(&ws->prb_rng, rng, errbuf, errlen))) return rc;
    }
    return 0;
}

static int wf_launch(sfw_stepper* h, WState* ws, int mode, int n_steps, int record_every, int ftab_stride, char* errbuf,
                     int errlen, int step0 = 0) {  // step0: first step of a later chunk (see sfw_step_run)
    WParams p{};
    p.n_sub = h->n_sub;
    p.L = h->L;
    p.BS = ws->BS;
    p.n_steps = n_steps;
    p.record_every = record_every;
    p.n_probe = h->n_probe;
    p.ftab_stride = ftab_stride;
    p.mode = mode;
    p.tag0 = ws->tag;
    p.dt = h->dt;
    p.dt2 = (float)(h->dt * h->dt);
    p.half = (float)((0.5 * h->dt) * h->dt);
    p.coef = ws->coef;
    p.W0 = ws->W[ws->cur];
    p.W1 = ws->W[ws->cur ^ 1];
    p.V0 = ws->V0;
    p.mbox = ws->mbox;
    p.cta_sub_ptr = h->cta_sub_ptr;
    p.nbr = h->nbr;
    p.src_ptr = h->src_ptr;
    p.src_ids = h->src_ids;
    p.src_vec = ws->src;
    p.src_voff = h->src_voff;
    p.ftab = ws->ftab + step0;
    p.prb_ptr = h->prb_ptr;
    p.prb_ids = h->prb_ids;
    p.prb_w = ws->prb;
    p.prb_woff = h->prb_woff;
    p.prb_rng = ws->prb_rng;
    p.rows = h->rows + (size_t)(step0 / record_every) * h->n_probe;
    p.norm_part = ws->norm + (size_t)step0 * h->grid * ws->nw;
    void* args[] = {&p};
    SFW_CUDA_TRY(cudaLaunchCooperativeKernel(ws->fn, dim3(h->grid), dim3(ws->nw * 32), args, ws->smem, h->stream));
    ws->tag += (unsigned int)(mode == 0 ? n_steps : 1);
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
    struct WScope { WScope() { ++sfw::g_wform_scope; } ~WScope() { --sfw::g_wform_scope; } } wscope_;
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
            if (!src) {  // stream-ordered: the legacy-stream cudaMemset would not order with h->stream
                if (ws->V0) cudaMemsetAsync(ws->V0, 0, n * 4, h->stream);
                continue;
            }
            if (!ws->V0 && (rc = dalloc(&ws->V0, n, errbuf, errlen))) return rc;
            dst = ws->V0;
        }
        if (!src) {
            cudaMemsetAsync(dst, 0, n * 4, h->stream);
            continue;
        }
        std::vector<double> out(n);
        if ((rc = wf_vectors(h, ws, h->n_sub, vs.data(), vo.data(), n, 0, src, out.data(), errbuf, errlen))) return rc;
        std::vector<float> f(out.begin(), out.end());
        sfw_h2d(dst, f.data(), n * 4);
    }
    if ((rc = wf_ensure(&ws->ftab, &ws->ftab_cap, std::max(1, h->n_src), errbuf, errlen))) return rc;
    if (h->n_src) {
        std::vector<float> f(profile0, profile0 + h->n_src);
        sfw_h2d(ws->ftab, f.data(), h->n_src * 4);
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
    if ((rc = wf_launch(h, ws, 1, 1, 1, 1, errbuf, errlen))) return rc;
    if (row0_out && h->n_probe)
        SFW_CUDA_TRY(cudaMemcpyAsync(row0_out, h->rows, h->n_probe * 8, cudaMemcpyDeviceToHost, h->stream));
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    return 0;
}

// |W| per step from the per-warp partials, summed in ascending partial order (one thread per step)
__global__ void k_wnorms(const double* __restrict__ part, int n_steps, long long nwg, double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_steps) return;
    double t = 0.0;
    for (long long c = 0; c < nwg; ++c) t += part[(size_t)k * nwg + c];
    out[k] = sqrt(t);
}

// n_steps fp32 W-form leapfrog steps.  Same table conventions as sfw_step_run; norms are |W| (the
// W-form invariant scale), rows are the physical probe values.  With limits (HOST [n_steps]) the
// growth detector runs in the library's norm path: the run is launched in chunks of <= 512 steps,
// each chunk's |W| is reduced on the device and checked while the next chunk computes, and no
// further chunk is launched once a step exceeds its limit (SFW_EINSTABLE, *bad_step = first
// failing step, 1-based); the state then has advanced at most one chunk past it.
extern "C" int sfw_wform_run(sfw_stepper* h, int n_steps, int record_every, const double* profile,
                             const double* limits, double* rows_out, double* norms_out, int* bad_step,
                             float* kernel_ms, char* errbuf, int errlen) {
    struct WScope { WScope() { ++sfw::g_wform_scope; } ~WScope() { --sfw::g_wform_scope; } } wscope_;
    WState* ws = g_wf.count(h) ? g_wf[h] : nullptr;
    if (bad_step) *bad_step = 0;
    if (!ws) return fail(SFW_ECONFIG, "call sfw_wform_setup first", errbuf, errlen);
    if (n_steps <= 0) return 0;
    if (record_every < 1) return fail(SFW_ECONFIG, "record_every must be >= 1", errbuf, errlen);
    if (h->n_src && !profile)
        return fail(SFW_ECONFIG, "a stepper with sources needs the f(t_k) profile table", errbuf, errlen);
    int rc = wf_ensure(&ws->ftab, &ws->ftab_cap, std::max(1LL, (long long)h->n_src * n_steps), errbuf, errlen);
    if (rc) return rc;
    if (h->n_src) {
        std::vector<float> f(profile, profile + (size_t)h->n_src * n_steps);
        sfw_h2d(ws->ftab, f.data(), f.size() * 4);
    }
    const long long nrec = n_steps / record_every;
    if (h->rows_cap < std::max(1LL, nrec * h->n_probe)) {
        if (h->rows) cudaFree(h->rows);
        h->rows = nullptr;
        if ((rc = dalloc(&h->rows, std::max(1LL, nrec * h->n_probe), errbuf, errlen))) return rc;
        h->rows_cap = std::max(1LL, nrec * h->n_probe);
    }
    const long long nwg = (long long)h->grid * ws->nw;
    if (ws->norm_cap < (long long)n_steps * nwg + n_steps) {
        if (ws->norm) cudaFree(ws->norm);
        ws->norm = nullptr;
        if ((rc = dalloc(&ws->norm, (size_t)n_steps * nwg + n_steps, errbuf, errlen))) return rc;
        ws->norm_cap = (long long)n_steps * nwg + n_steps;
    }
    double* dnorm = ws->norm + (size_t)n_steps * nwg;  // reduced |W| per step
    // large probe-row downloads overlap later chunks of the run (chunk_plan, as sfw_step_run);
    // with a growth limit, chunks are also capped at 512 steps (whole record intervals)
    std::vector<long long> plan = chunk_plan(nrec, nrec * h->n_probe * 8, rows_out != nullptr);
    if (limits && nrec > 0) {
        const long long cap = std::max(1LL, 512LL / record_every);
        std::vector<long long> fine{0};
        for (size_t c = 1; c < plan.size(); ++c)
            for (long long v = fine.back() + cap; ; v += cap) {
                if (v >= plan[c]) {
                    fine.push_back(plan[c]);
                    break;
                }
                fine.push_back(v);
            }
        plan.swap(fine);
    }
    const int n_chunks = (int)plan.size() - 1;
    if (n_chunks > 1 && !h->dstream) SFW_CUDA_TRY(cudaStreamCreateWithFlags(&h->dstream, cudaStreamNonBlocking));
    if (n_chunks > 1 && rows_out) SFW_CUDA_TRY(ensure_row_staging(h, plan, h->n_probe));
    std::vector<cudaEvent_t> evs;
    std::vector<int> bounds;  // first step of each launched chunk, then n_steps
    std::vector<double> nrm(n_steps);
    int bad = 0, checked = 0;  // steps [0, checked) verified against limits
    auto check_upto = [&](int upto) -> cudaError_t {  // host copy + check of steps [checked, upto)
        if (upto <= checked) return cudaSuccess;
        cudaError_t e = cudaMemcpy(nrm.data() + checked, dnorm + checked, (size_t)(upto - checked) * 8,
                                   cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return e;
        for (int k = checked; k < upto && !bad; ++k)
            if (!(nrm[k] <= limits[k])) bad = k + 1;  // NaN counts as divergence
        checked = upto;
        return cudaSuccess;
    };
    SFW_CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
    for (int c = 0; c < n_chunks; ++c) {
        const long long r0 = plan[c], r1 = plan[c + 1];
        const int s0 = (int)(r0 * record_every);
        const int s1 = (c == n_chunks - 1) ? n_steps : (int)(r1 * record_every);
        if ((rc = wf_launch(h, ws, 0, s1 - s0, record_every, n_steps, errbuf, errlen, s0))) return rc;
        ws->cur ^= ((s1 - s0) & 1);
        k_wnorms<<<(s1 - s0 + 127) / 128, 128, 0, h->stream>>>(ws->norm + (size_t)s0 * nwg, s1 - s0, nwg, dnorm + s0);
        bounds.push_back(s0);
        cudaEvent_t e;
        SFW_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        SFW_CUDA_TRY(cudaEventRecord(e, h->stream));
        evs.push_back(e);
        if (limits && c >= 1) {  // check the previous chunk while this one computes
            SFW_CUDA_TRY(cudaEventSynchronize(evs[c - 1]));
            SFW_CUDA_TRY(check_upto(s0));
            if (bad) break;
        }
    }
    bounds.push_back(n_steps);
    SFW_CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
    const int launched = (int)evs.size();
    if (launched > 1 && rows_out) {  // rows of the launched chunks (the pageable norm copy blocks)
        std::vector<long long> lplan(plan.begin(), plan.begin() + launched + 1);
        SFW_CUDA_TRY(download_rows_overlapped(h, lplan, evs, h->rows, rows_out, h->n_probe));
    }
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    const int done = (launched == n_chunks) ? n_steps : bounds[launched];
    if (launched == 1 && rows_out && nrec * h->n_probe > 0)
        SFW_CUDA_TRY(cudaMemcpy(rows_out, h->rows, (size_t)nrec * h->n_probe * 8, cudaMemcpyDeviceToHost));
    if (limits && !bad) SFW_CUDA_TRY(check_upto(done));
    if (!limits || checked < done)
        SFW_CUDA_TRY(cudaMemcpy(nrm.data(), dnorm, (size_t)done * 8, cudaMemcpyDeviceToHost));
    if (kernel_ms) cudaEventElapsedTime(kernel_ms, h->ev0, h->ev1);
    if (norms_out) std::memcpy(norms_out, nrm.data(), (size_t)done * 8);
    if (bad) {
        if (bad_step) *bad_step = bad;
        char msg[256];
        snprintf(msg, sizeof msg, "coupled stepping diverged: |W| = %.3e exceeds %.3e", nrm[bad - 1], limits[bad - 1]);
        return fail(SFW_EINSTABLE, msg, errbuf, errlen);
    }
    return 0;
}

// W-form state as U-form (U_j = G_j W_j), fp64, HOST concat.
extern "C" int sfw_wform_state(sfw_stepper* h, double* u_curr, double* u_prev, char* errbuf, int errlen) {
    struct WScope { WScope() { ++sfw::g_wform_scope; } ~WScope() { --sfw::g_wform_scope; } } wscope_;
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
    struct WScope { WScope() { ++sfw::g_wform_scope; } ~WScope() { --sfw::g_wform_scope; } } wscope_;
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
    struct WScope { WScope() { ++sfw::g_wform_scope; } ~WScope() { --sfw::g_wform_scope; } } wscope_;
    if (!g_wf.count(h)) return 0;
    WState* ws = g_wf[h];
    void* ptrs[] = {ws->coef, ws->W[0], ws->W[1], ws->V0, ws->mbox, ws->src, ws->prb, ws->ftab, ws->prb_rng,
                    ws->norm, ws->first_blk};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    delete ws;
    g_wf.erase(h);
    return 0;
}
