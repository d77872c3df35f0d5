// Multi-shot stepping (BASELINE config 4): S independent wavefields advanced in
// one persistent launch.  The reference runs one CoupledStepper per shot
// (stepper.py:144-449 with a single SourceTerm); here the
// state of a subdomain layer is a w x S block and every chain block product
// Gamma_j X / Gamma-hat_j X is a (w x w)(w x S) fp64 GEMM on the DMMA pipe
// (mma.sync.m8n8k4.f64).
//
// Block storage: the lower 8 x 8 tiles (I >= K) of the padded w x w symmetric
// block, each tile stored in DMMA A-fragment order (half h, lane l) ->
// element (l/4, 4h + l%4).  Warp I owns output row-tile I and applies tile
// (I,K) for K <= I and the transpose of tile (K,I) for K > I, so the symmetric
// block is streamed once (+20% bytes over w(w+1)/2 for w = 54) and no
// cross-warp reduction is needed.
//
// One CTA walks its subdomains; per step:
//   phase A  flux_1, acc_1 = Gamma-hat_1 flux_1 of every subdomain (published)
//   phase B  layers 2..L by a sliding window (U_j, U_{j+1}, flux_{j-1} in SMEM),
//            leapfrog fused into the Gamma-hat epilogue
//   phase C  (after the neighbour flags) layer-1 face coupling + leapfrog,
//            per-shot |U|^2 partials and probe rows
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "sfw_common.cuh"
#include "sfw_linalg.cuh"
#include "sfw_step_internal.cuh"

namespace sfw {

__host__ __device__ inline int ms_packed_pos(int m, int row, int col) {
    // identical to packed_pos() in sfw_step.cu (6-group packed symmetric layout)
    if (row < col) {
        int t = row;
        row = col;
        col = t;
    }
    int I = row / m, K = col / m, r = row % m, c = col % m;
    if (I != K) {
        int t = I * (I - 1) / 2 + K;
        int q = (c - r + m) % m;
        int e = q * m + r;
        return e * 15 + t;
    }
    int d = r - c;
    int e = 0;
    for (int dd = 0; dd < d; ++dd) e += m - dd;
    e += c;
    return 15 * m * m + e * 6 + I;
}

// 6-group packed blocks -> fragment-ordered lower 8x8 tiles
__global__ void k_tilepack(const double* __restrict__ packed, int BS, int m, int RT, int TB,
                           double* __restrict__ out, long long n_blocks) {
    const long long b = blockIdx.x;
    if (b >= n_blocks) return;
    const int w = 6 * m;
    const double* src = packed + b * BS;
    double* dst = out + b * TB;
    const int ntl = RT * (RT + 1) / 2;
    for (int idx = threadIdx.x; idx < ntl * 64; idx += blockDim.x) {
        const int t = idx / 64, within = idx % 64;
        int I = 0;
        while ((I + 1) * (I + 2) / 2 <= t) ++I;
        const int K = t - I * (I + 1) / 2;
        const int h = within / 32, l = within % 32;
        const int r = l >> 2, c = 4 * h + (l & 3);
        const int row = I * 8 + r, col = K * 8 + c;
        dst[idx] = (row < w && col < w) ? src[ms_packed_pos(m, row, col)] : 0.0;
    }
}

struct MsParams {
    int n_sub, L, W, WP, RT, TB, S, n_steps, record_every, n_probe, ftab_stride;
    long long K;  // L*W
    double dt2;
    const double* tcoef;
    double* U0;
    double* U1;
    double* flux;   // [n_sub][W][S] layer-1 flux (face mailbox), double-buffered by parity
    double* acc1;   // [n_sub][W][S]
    const int* nbr;
    const int* mass_idx;
    const double* mass;
    const int* cta_sub_ptr;
    const int* shot_sub;   // [S] source subdomain of each shot (-1: none)
    const double* shot_vec;
    const long long* shot_voff;
    const double* ftab;    // [S][n_steps]
    const int* prb_ptr;
    const int* prb_ids;
    const int* prb_tap;
    const double* prb_w;
    const long long* prb_woff;
    double* rows;          // [n_rec][n_probe][S]
    double* norm_part;     // [n_steps][grid][S]
    unsigned int* flags;
    const int* ncta_ptr;
    const int* ncta;
    int evict_first;
};

constexpr int MS_NW = 16;  // warp = (row tile I = warp/2, column half = warp%2)
constexpr int MS_NS = 3;   // chain-block (coefficient) TMA stages
constexpr int MS_NSS = 4;  // state-block TMA stages

// Y(row-tile I, column tiles c0..c0+CTW-1) = Gamma X, X in smem [WP][LDX]; acc[ct][2]
template <int CTW>
__device__ __forceinline__ void ms_matmul(const double* __restrict__ tiles, const double* __restrict__ Xs, int LDX,
                                          int RT, int I, int c0, int lane, const int (&tr)[2], double (&acc)[CTW][2]) {
#pragma unroll
    for (int ct = 0; ct < CTW; ++ct) acc[ct][0] = acc[ct][1] = 0.0;
    for (int Kt = 0; Kt < RT; ++Kt) {
        const bool normal = (I >= Kt);
        const int t = normal ? (I * (I + 1) / 2 + Kt) : (Kt * (Kt + 1) / 2 + I);
        const double* tp = tiles + t * 64;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double a = tp[normal ? (h * 32 + lane) : tr[h]];
            const double* xr = Xs + (Kt * 8 + 4 * h + (lane & 3)) * LDX + c0 * 8 + (lane >> 2);
#pragma unroll
            for (int ct = 0; ct < CTW; ++ct) dmma8x8x4(acc[ct], a, xr[ct * 8]);
        }
    }
}

// State-block stream of one CTA per step (each block = one layer of one subdomain, W x S):
//   A: for s: U_0, U_1 (current)
//   B: for s: Fx (layer-1 flux of phase A), U_1, then j = 1..L-1: [U_{j+1} if j+1 < L], Uprev_j
//   C: for s: U_0, Uprev_0
// Gates: A blocks of step k are issued only after step k-1 finished (they are its
// output); B/C blocks only after phase A of step k (Fx is its output).
struct MsStream {
    int ns, L;
    __device__ __forceinline__ int per_step() const { return ns * (2 * L + 3); }
    __device__ __forceinline__ int endA() const { return 2 * ns; }
    // returns global offset (in doubles) of block at position p; phase in *ph
    __device__ __forceinline__ long long where(int p, int s0, long long WS, long long KS, const MsParams& prm,
                                               int cb, int* ph) const {
        const double* cur = cb ? prm.U1 : prm.U0;
        const double* prv = cb ? prm.U0 : prm.U1;
        (void)cur;
        (void)prv;
        if (p < 2 * ns) {
            *ph = 0;
            const int sl = p >> 1;
            return (long long)(s0 + sl) * KS + (p & 1) * WS + ((long long)cb << 62);  // tag: buffer in high bits
        }
        p -= 2 * ns;
        const int nb = 2 * L - 1;
        if (p < ns * nb) {
            *ph = 1;
            const int sl = p / nb, r = p % nb;
            if (r == 0) return -1 - (long long)(s0 + sl);  // Fx block: negative tag
            if (r == 1) return (long long)(s0 + sl) * KS + 1 * WS + ((long long)cb << 62);
            const int rp = r - 2;
            if (rp < 2 * (L - 2)) {
                const int j = 1 + rp / 2;
                if ((rp & 1) == 0) return (long long)(s0 + sl) * KS + (j + 1) * WS + ((long long)cb << 62);
                return (long long)(s0 + sl) * KS + j * WS + ((long long)(cb ^ 1) << 62);
            }
            return (long long)(s0 + sl) * KS + (L - 1) * WS + ((long long)(cb ^ 1) << 62);
        }
        p -= ns * nb;
        *ph = 2;
        const int sl = p >> 1;
        return (long long)(s0 + sl) * KS + ((long long)((p & 1) ? (cb ^ 1) : cb) << 62);
    }
};

template <int S>
__global__ void __launch_bounds__((MS_NW + 1) * 32, 1) k_step_ms(const MsParams p) {
    constexpr int CTW = S / 16;  // column tiles per warp (two warps share a row tile)
    constexpr int LDX = S + 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = p.W, WP = p.WP, RT = p.RT, L = p.L, TB = p.TB;
    const long long K = p.K;
    const long long WS = (long long)W * S, KS = K * S;
    double* cst = reinterpret_cast<double*>(smem_raw);   // MS_NS * TB
    double* sst = cst + (size_t)MS_NS * TB;              // MS_NSS * WS
    double* Xs = sst + (size_t)MS_NSS * WS;              // [WP][LDX]
    double* Fa = Xs + WP * LDX;
    double* Fb = Fa + WP * LDX;
    double* Ua_ = Fb + WP * LDX;
    double* Ub_ = Ua_ + WP * LDX;
    double* red = Ub_ + WP * LDX;                        // [MS_NW][S]
    uint64_t* cfull = reinterpret_cast<uint64_t*>(red + MS_NW * S);
    uint64_t* cempty = cfull + MS_NS;
    uint64_t* sfull = cempty + MS_NS;
    uint64_t* sempty = sfull + MS_NSS;
    int* ssub = reinterpret_cast<int*>(sempty + MS_NSS);
    volatile int* gate_sh = ssub + S;

    for (int q = threadIdx.x; q < S; q += blockDim.x) ssub[q] = p.shot_sub[q];
    if (threadIdx.x == 0) {
        for (int i = 0; i < MS_NS; ++i) {
            mbar_init(&cfull[i], 1);
            mbar_init(&cempty[i], 1);
        }
        for (int i = 0; i < MS_NSS; ++i) {
            mbar_init(&sfull[i], 1);
            mbar_init(&sempty[i], 1);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 5 * WP * LDX; i += blockDim.x) Xs[i] = 0.0;  // zero pads of all operand buffers
    const int s0 = p.cta_sub_ptr[blockIdx.x], s1 = p.cta_sub_ptr[blockIdx.x + 1];
    const int ns = s1 - s0;
    const MsStream sm{ns, L};
    const int sper = sm.per_step();
    if (threadIdx.x == 0) *gate_sh = sm.endA();
    __syncthreads();

    // ======== producer warp: TMA streams of chain blocks and state blocks ========
    if (warp == MS_NW) {
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_first();
            const uint64_t pol_state = l2_policy_evict_last();
            const int cper = ns * 2 * L;
            const int ctotal = cper * p.n_steps;
            const int stotal = sper * p.n_steps;
            const uint32_t sbytes = (uint32_t)(WS * 8), cbytes = (uint32_t)TB * 8u;
            int c_iss = 0, s_iss = 0;
            int cpos = 0;  // position within the step of the coefficient stream
            while (c_iss < ctotal || s_iss < stotal) {
                bool did = false;
                if (c_iss < ctotal) {
                    const int st = c_iss % MS_NS;
                    if (mbar_test_wait(&cempty[st], (uint32_t)(((c_iss / MS_NS) & 1) ^ 1))) {
                        long long blk;
                        if (cpos < 2 * ns) {
                            blk = ((long long)(s0 + cpos / 2) * L) * 2 + (cpos & 1);
                        } else {
                            const int r = cpos - 2 * ns;
                            const int sl = r / (2 * (L - 1)), rr = r % (2 * (L - 1));
                            blk = ((long long)(s0 + sl) * L + 1 + rr / 2) * 2 + (rr & 1);
                        }
                        mbar_arrive_expect_tx(&cfull[st], cbytes);
                        bulk_g2s(cst + (size_t)st * TB, p.tcoef + blk * TB, cbytes, &cfull[st], pol);
                        ++c_iss;
                        if (++cpos == cper) cpos = 0;
                        did = true;
                    }
                }
                if (s_iss < stotal && s_iss < *gate_sh) {
                    const int st = s_iss % MS_NSS;
                    if (mbar_test_wait(&sempty[st], (uint32_t)(((s_iss / MS_NSS) & 1) ^ 1))) {
                        const int step = s_iss / sper;
                        const int cb = step & 1;
                        int ph;
                        const long long tag = sm.where(s_iss % sper, s0, WS, KS, p, cb, &ph);
                        const double* src;
                        if (tag < 0) {
                            src = p.flux + ((size_t)((step + 1) & 1) * p.n_sub + (-1 - tag)) * WS;
                        } else {
                            const int buf = (int)((unsigned long long)tag >> 62);
                            src = (buf ? p.U1 : p.U0) + (tag & ((1LL << 62) - 1));
                        }
                        fence_proxy_async();
                        mbar_arrive_expect_tx(&sfull[st], sbytes);
                        bulk_g2s(sst + (size_t)st * WS, src, sbytes, &sfull[st], pol_state);
                        ++s_iss;
                        did = true;
                    }
                }
            }
        }
        return;
    }

    // ======== compute warps ========
    int tr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = 4 * h + (lane & 3), c = lane >> 2;
        tr[h] = (c >> 2) * 32 + r * 4 + (c & 3);
    }
    int c_con = 0, s_con = 0;
    auto csync = []() { asm volatile("bar.sync 1, %0;" ::"r"(MS_NW * 32) : "memory"); };
    auto c_acquire = [&]() -> const double* {
        const int st = c_con % MS_NS;
        mbar_wait(&cfull[st], (uint32_t)((c_con / MS_NS) & 1));
        return cst + (size_t)st * TB;
    };
    auto s_acquire = [&]() -> const double* {
        const int st = s_con % MS_NSS;
        mbar_wait(&sfull[st], (uint32_t)((s_con / MS_NSS) & 1));
        return sst + (size_t)st * WS;
    };
    auto released = [&](int nc, int nsr) {  // caller has done csync(): every compute warp is done with them
        if (threadIdx.x == 0) {
            for (int i = 0; i < nc; ++i) mbar_arrive(&cempty[(c_con + i) % MS_NS]);
            for (int i = 0; i < nsr; ++i) mbar_arrive(&sempty[(s_con + i) % MS_NSS]);
        }
        c_con += nc;
        s_con += nsr;
    };
    auto open_gate = [&](int pos) {  // after csync(): state written so far may be streamed
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            *gate_sh = pos;
        }
    };

    const int I = warp >> 1, c0 = (warp & 1) * CTW;
    const int orow = I * 8 + (lane >> 2);
    const bool active = (I < RT) && (orow < W);
    double sq[CTW][2];
    const double dt2 = p.dt2;
    const int M = W / 6;

    for (int k = 1; k <= p.n_steps; ++k) {
        const int par = k & 1;
        const int cb = (k - 1) & 1;
        double* Un = cb ? p.U0 : p.U1;
        double* fx = p.flux + (size_t)par * p.n_sub * WS;
        const int kk = k - 1;
        const int base = (k - 1) * sper;
#pragma unroll
        for (int ct = 0; ct < CTW; ++ct) sq[ct][0] = sq[ct][1] = 0.0;

        // ---------------- phase A: flux_1 and acc_1 --------------------------------
        for (int sl = 0; sl < ns; ++sl) {
            const int s = s0 + sl;
            const double* u0 = s_acquire();
            ++s_con;  // consume order: U_0, U_1 (released together below)
            const double* u1 = s_acquire();
            --s_con;
            for (int idx = threadIdx.x; idx < W * S; idx += MS_NW * 32) {
                const int r = idx / S, c = idx % S;
                Xs[r * LDX + c] = u1[idx] - u0[idx];
            }
            csync();
            released(0, 2);
            double acc[CTW][2];
            const double* tl = c_acquire();
            if (I < RT) ms_matmul<CTW>(tl, Xs, LDX, RT, I, c0, lane, tr, acc);
            if (active)
#pragma unroll
                for (int ct = 0; ct < CTW; ++ct)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = (c0 + ct) * 8 + (lane & 3) * 2 + e;
                        Fa[orow * LDX + col] = acc[ct][e];
                        fx[((size_t)s * W + orow) * S + col] = acc[ct][e];
                    }
            csync();
            released(1, 0);
            tl = c_acquire();
            if (I < RT) ms_matmul<CTW>(tl, Fa, LDX, RT, I, c0, lane, tr, acc);
            if (active)
#pragma unroll
                for (int ct = 0; ct < CTW; ++ct)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        p.acc1[((size_t)s * W + orow) * S + (c0 + ct) * 8 + (lane & 3) * 2 + e] = acc[ct][e];
            csync();
            released(1, 0);
        }
        open_gate(base + sper);  // phase B/C blocks of this step may now stream (Fx written)
        if (threadIdx.x == 0) flag_publish(p.flags, (unsigned int)k);

        // ---------------- phase B: layers 2..L (sliding window) ------------------------
        for (int sl = 0; sl < ns; ++sl) {
            const int s = s0 + sl;
            double* un = Un + (size_t)s * KS;
            {
                const double* fxs = s_acquire();
                ++s_con;
                const double* u1 = s_acquire();
                --s_con;
                for (int idx = threadIdx.x; idx < W * S; idx += MS_NW * 32) {
                    const int r = idx / S, c = idx % S;
                    Fb[r * LDX + c] = fxs[idx];
                    Ua_[r * LDX + c] = u1[idx];
                }
                csync();
                released(0, 2);
            }
            double* Fc = Fa;   // flux_j (new)
            double* Fo = Fb;   // flux_{j-1}
            double* Ua = Ua_;  // U_j
            double* Ub = Ub_;  // U_{j+1}
            for (int j = 1; j < L; ++j) {
                if (j + 1 < L) {
                    const double* un1 = s_acquire();
                    for (int idx = threadIdx.x; idx < W * S; idx += MS_NW * 32) {
                        const int r = idx / S, c = idx % S;
                        const double v = un1[idx];
                        Ub[r * LDX + c] = v;
                        Xs[r * LDX + c] = v - Ua[r * LDX + c];
                    }
                    csync();
                    released(0, 1);
                } else {
                    for (int idx = threadIdx.x; idx < W * S; idx += MS_NW * 32) {
                        const int r = idx / S, c = idx % S;
                        Xs[r * LDX + c] = 0.0 - Ua[r * LDX + c];
                    }
                    csync();
                }
                double acc[CTW][2];
                const double* tl = c_acquire();
                if (I < RT) ms_matmul<CTW>(tl, Xs, LDX, RT, I, c0, lane, tr, acc);
                if (active)
#pragma unroll
                    for (int ct = 0; ct < CTW; ++ct)
#pragma unroll
                        for (int e = 0; e < 2; ++e) Fc[orow * LDX + (c0 + ct) * 8 + (lane & 3) * 2 + e] = acc[ct][e];
                csync();
                released(1, 0);
                for (int idx = threadIdx.x; idx < W * S; idx += MS_NW * 32) {
                    const int r = idx / S, c = idx % S;
                    Xs[r * LDX + c] = Fc[r * LDX + c] - Fo[r * LDX + c];
                }
                csync();
                const double* uo = s_acquire();  // Uprev_j
                tl = c_acquire();
                if (I < RT) ms_matmul<CTW>(tl, Xs, LDX, RT, I, c0, lane, tr, acc);
                if (active) {
#pragma unroll
                    for (int ct = 0; ct < CTW; ++ct)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int col = (c0 + ct) * 8 + (lane & 3) * 2 + e;
                            double tot = acc[ct][e];
                            if (ssub[col] == s) {
                                const double term =
                                    __dmul_rn(p.shot_vec[p.shot_voff[col] + (size_t)j * W + orow],
                                              p.ftab[(size_t)col * p.ftab_stride + kk]);
                                tot = __dadd_rn(tot, term);
                            }
                            const double v = __dadd_rn(__dsub_rn(__dmul_rn(2.0, Ua[orow * LDX + col]),
                                                                 uo[orow * S + col]),
                                                       __dmul_rn(dt2, tot));
                            un[((size_t)j * W + orow) * S + col] = v;
                            sq[ct][e] = fma(v, v, sq[ct][e]);
                        }
                }
                csync();
                released(1, 1);
                double* t = Fc;
                Fc = Fo;
                Fo = t;
                t = Ua;
                Ua = Ub;
                Ub = t;
            }
        }

        // ---------------- neighbour flags, then phase C --------------------------------
        if (warp == 0)
            flags_wait(p.flags, p.ncta + p.ncta_ptr[blockIdx.x], p.ncta_ptr[blockIdx.x + 1] - p.ncta_ptr[blockIdx.x],
                       (unsigned int)k, lane);
        csync();
        for (int sl = 0; sl < ns; ++sl) {
            const int s = s0 + sl;
            double* un = Un + (size_t)s * KS;
            const double* u0 = s_acquire();
            ++s_con;
            const double* uo = s_acquire();
            --s_con;
            if (active) {
                const int f = orow / M, r = orow % M;
                const int nb = p.nbr[s * 6 + f];
#pragma unroll
                for (int ct = 0; ct < CTW; ++ct)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = (c0 + ct) * 8 + (lane & 3) * 2 + e;
                        double a;
                        if (nb >= 0) {
                            const double* mx = p.mass + (size_t)p.mass_idx[s * 6 + f] * M * M + r * M;
                            const double* own = fx + ((size_t)s * W + f * M) * S + col;
                            const double* oth = fx + ((size_t)nb * W + (f ^ 1) * M) * S + col;
                            a = 0.0;
                            for (int c = 0; c < M; ++c) a = fma(mx[c], __dadd_rn(own[c * S], oth[c * S]), a);
                        } else {
                            a = p.acc1[((size_t)s * W + orow) * S + col];
                        }
                        if (ssub[col] == s) {
                            const double term = __dmul_rn(p.shot_vec[p.shot_voff[col] + orow],
                                                          p.ftab[(size_t)col * p.ftab_stride + kk]);
                            a = __dadd_rn(a, term);
                        }
                        const size_t g = (size_t)orow * S + col;
                        const double v = __dadd_rn(__dsub_rn(__dmul_rn(2.0, u0[g]), uo[g]), __dmul_rn(dt2, a));
                        un[g] = v;
                        sq[ct][e] = fma(v, v, sq[ct][e]);
                    }
            }
            csync();
            released(0, 2);
        }
        // per-shot |U|^2: lanes sharing (lane & 3) own the same columns -> fixed-order reduction
#pragma unroll
        for (int ct = 0; ct < CTW; ++ct)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double v = sq[ct][e];
                for (int o = 4; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane < 4) red[I * S + (c0 + ct) * 8 + lane * 2 + e] = v;  // each (row tile, column) once
            }
        csync();
        for (int q = threadIdx.x; q < S; q += MS_NW * 32) {
            double t = 0.0;
            for (int i2 = 0; i2 < MS_NW / 2; ++i2) t += red[i2 * S + q];
            p.norm_part[((size_t)kk * gridDim.x + blockIdx.x) * S + q] = t;
        }
        if (k % p.record_every == 0 && p.rows) {
            const long long row = k / p.record_every - 1;
            for (int s = s0; s < s1; ++s) {
                const double* us = Un + (size_t)s * KS;
                for (int pq = p.prb_ptr[s] + warp; pq < p.prb_ptr[s + 1]; pq += MS_NW) {
                    const int pid = p.prb_ids[pq];
                    const int tap = p.prb_tap[pid];
                    for (int q = lane; q < S; q += 32) {
                        double val;
                        if (tap >= 0) {
                            val = us[(size_t)tap * S + q];
                        } else {
                            const double* wv = p.prb_w + p.prb_woff[pid];
                            val = 0.0;
                            for (long long i = 0; i < K; ++i) val = fma(wv[i], us[i * S + q], val);
                        }
                        p.rows[(row * p.n_probe + pid) * S + q] = val;
                    }
                }
            }
        }
        csync();
        open_gate(k * sper + sm.endA());  // next step's phase A inputs are written
    }
}

// shots start from rest (u0 = v0 = 0): U_curr = 0, U_prev = ((0.5 dt) dt) (vec_q f_q(0))  (stepper.py:347-353)
__global__ void k_ms_init(double* U0, double* U1, long long total, int S, const int* shot_sub,
                          const double* shot_vec, const long long* shot_voff, const double* f0, double half,
                          long long K) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(i % S);
        const long long rest = i / S;
        const long long s = rest / K, idx = rest % K;
        U0[i] = 0.0;
        double v = 0.0;
        if (shot_sub[q] == s) v = __dmul_rn(half, __dmul_rn(shot_vec[shot_voff[q] + idx], f0[q]));
        U1[i] = v;
    }
}

__global__ void k_ms_norms(const double* __restrict__ part, int n_steps, int n_cta, int S, double* __restrict__ out) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= (long long)n_steps * S) return;
    const int k = (int)(i / S), q = (int)(i % S);
    double t = 0.0;
    for (int c = 0; c < n_cta; ++c) t += part[((size_t)k * n_cta + c) * S + q];
    out[i] = sqrt(t);
}

}  // namespace sfw

using namespace sfw;

static int ms_ensure(double** p, long long* cap, long long need, char* errbuf, int errlen) {
    if (*cap >= need && *p) return 0;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    int rc = dalloc(p, need, errbuf, errlen);
    if (!rc) *cap = need;
    return rc;
}

// Enable multi-shot mode on a stepper: S = n_shots independent wavefields, shot q
// forced by vector shot_vec[q] (length L*w of subdomain shot_sub[q]).  S must be 32.
extern "C" int sfw_shots_setup(sfw_stepper* h, int n_shots, const int* shot_sub, const double* shot_vec,
                               char* errbuf, int errlen) {
    if (n_shots != 32) return fail(SFW_ECONFIG, "multi-shot stepping supports exactly 32 shots", errbuf, errlen);
    if (!h->uniform) return fail(SFW_ECONFIG, "multi-shot stepping needs one layer count for all models", errbuf, errlen);
    const int S = n_shots, W = h->W, L = h->L;
    const int WP = (W + 7) & ~7, RT = WP / 8;
    h->TB = RT * (RT + 1) / 2 * 64;
    h->n_shots = S;
    int rc = 0;
    if (!h->tcoef) {
        if ((rc = dalloc(&h->tcoef, (size_t)h->n_blocks * h->TB, errbuf, errlen))) return rc;
        k_tilepack<<<(unsigned)h->n_blocks, 256, 0, h->stream>>>(h->coef, h->BS, h->m, RT, h->TB, h->tcoef,
                                                                 h->n_blocks);
    }
    const size_t st = (size_t)h->n_sub * L * W * S;
    for (int b = 0; b < 2; ++b)
        if (!h->UM[b] && (rc = dalloc(&h->UM[b], st, errbuf, errlen))) return rc;
    if (!h->mfb && (rc = dalloc(&h->mfb, (size_t)2 * h->n_sub * W * S, errbuf, errlen))) return rc;
    if (!h->macc1 && (rc = dalloc(&h->macc1, (size_t)h->n_sub * W * S, errbuf, errlen))) return rc;
    std::vector<long long> voff(S);
    long long vt = 0;
    for (int q = 0; q < S; ++q) {
        const int s = shot_sub[q];
        if (s < -1 || s >= h->n_sub) return fail(SFW_ECONFIG, "shot source subdomain has no model", errbuf, errlen);
        voff[q] = vt;
        if (s >= 0) vt += h->soff[s + 1] - h->soff[s];
    }
    std::vector<int> ss(shot_sub, shot_sub + S);
    std::vector<double> sv(shot_vec, shot_vec + std::max(vt, 1LL));
    if (h->shot_sub) cudaFree(h->shot_sub);
    if (h->shot_voff) cudaFree(h->shot_voff);
    if (h->shot_vec) cudaFree(h->shot_vec);
    h->shot_sub = nullptr;
    h->shot_voff = nullptr;
    h->shot_vec = nullptr;
    if ((rc = upload(&h->shot_sub, ss, errbuf, errlen))) return rc;
    if ((rc = upload(&h->shot_voff, voff, errbuf, errlen))) return rc;
    if ((rc = upload(&h->shot_vec, sv, errbuf, errlen))) return rc;
    h->shot_smem = (int)(8 * ((size_t)MS_NS * h->TB + (size_t)MS_NSS * W * S + 5 * (size_t)WP * (S + 4) +
                              MS_NW * S + 2 * MS_NS + 2 * MS_NSS) + 4 * S + 64);
    if (L < 2) return fail(SFW_ECONFIG, "multi-shot stepping needs at least 2 layers", errbuf, errlen);
    SFW_CUDA_TRY(cudaFuncSetAttribute((const void*)k_step_ms<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      h->shot_smem));
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    return 0;
}

// Run n_steps from rest for all shots.  profile: HOST [S][n_steps] f_q(t_k), t_k = k dt;
// profile0: HOST [S] f_q(0).  rows_out: HOST [n_steps/record_every][n_probe][S] (or NULL);
// norms_out: HOST [n_steps][S] (or NULL); *kernel_ms: CUDA-event time of the launch.
extern "C" int sfw_shots_run(sfw_stepper* h, int n_steps, int record_every, const double* profile0,
                             const double* profile, double* rows_out, double* norms_out, float* kernel_ms,
                             char* errbuf, int errlen) {
    if (!h->n_shots) return fail(SFW_ECONFIG, "call sfw_shots_setup first", errbuf, errlen);
    if (n_steps <= 0) return 0;
    if (record_every < 1) return fail(SFW_ECONFIG, "record_every must be >= 1", errbuf, errlen);
    const int S = h->n_shots, W = h->W, L = h->L;
    const int WP = (W + 7) & ~7, RT = WP / 8;
    int rc = ms_ensure(&h->shot_ftab, &h->shot_ftab_cap, (long long)S * n_steps + S, errbuf, errlen);
    if (rc) return rc;
    SFW_CUDA_TRY(cudaMemcpyAsync(h->shot_ftab, profile, (size_t)S * n_steps * 8, cudaMemcpyHostToDevice, h->stream));
    SFW_CUDA_TRY(cudaMemcpyAsync(h->shot_ftab + (size_t)S * n_steps, profile0, (size_t)S * 8, cudaMemcpyHostToDevice,
                                 h->stream));
    const long long nrec = n_steps / record_every;
    if ((rc = ms_ensure(&h->mrows, &h->mrows_cap, std::max(1LL, nrec * h->n_probe * S), errbuf, errlen))) return rc;
    if ((rc = ms_ensure(&h->mnorm, &h->mnorm_cap, (long long)n_steps * h->grid * S + (long long)n_steps * S, errbuf,
                        errlen)))
        return rc;
    const long long total = (long long)h->n_sub * L * W * S;
    const double half = (0.5 * h->dt) * h->dt;
    k_ms_init<<<1184, 256, 0, h->stream>>>(h->UM[0], h->UM[1], total, S, h->shot_sub, h->shot_vec, h->shot_voff,
                                           h->shot_ftab + (size_t)S * n_steps, half, (long long)L * W);
    SFW_CUDA_TRY(cudaMemsetAsync(h->bar, 0, sizeof(unsigned int) * h->grid, h->stream));
    MsParams p{};
    p.n_sub = h->n_sub;
    p.L = L;
    p.W = W;
    p.WP = WP;
    p.RT = RT;
    p.TB = h->TB;
    p.S = S;
    p.n_steps = n_steps;
    p.record_every = record_every;
    p.n_probe = h->n_probe;
    p.ftab_stride = n_steps;
    p.K = (long long)L * W;
    p.dt2 = h->dt * h->dt;
    p.tcoef = h->tcoef;
    p.U0 = h->UM[0];
    p.U1 = h->UM[1];
    p.flux = h->mfb;
    p.acc1 = h->macc1;
    p.nbr = h->nbr;
    p.mass_idx = h->mass_idx;
    p.mass = h->mass;
    p.cta_sub_ptr = h->cta_sub_ptr;
    p.shot_sub = h->shot_sub;
    p.shot_vec = h->shot_vec;
    p.shot_voff = h->shot_voff;
    p.ftab = h->shot_ftab;
    p.prb_ptr = h->prb_ptr;
    p.prb_ids = h->prb_ids;
    p.prb_tap = h->prb_tap;
    p.prb_w = h->prb_w;
    p.prb_woff = h->prb_woff;
    p.rows = h->mrows;
    p.norm_part = h->mnorm;
    p.flags = h->bar;
    p.ncta_ptr = h->ncta_ptr;
    p.ncta = h->ncta;
    p.evict_first = 1;
    void* args[] = {&p};
    SFW_CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
    SFW_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_step_ms<32>, dim3(h->grid), dim3((MS_NW + 1) * 32), args,
                                             h->shot_smem, h->stream));
    SFW_CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
    double* dn = h->mnorm + (size_t)n_steps * h->grid * S;
    k_ms_norms<<<(unsigned)((n_steps * S + 255) / 256), 256, 0, h->stream>>>(h->mnorm, n_steps, h->grid, S, dn);
    if (norms_out)
        SFW_CUDA_TRY(cudaMemcpyAsync(norms_out, dn, (size_t)n_steps * S * 8, cudaMemcpyDeviceToHost, h->stream));
    if (rows_out && nrec * h->n_probe > 0)
        SFW_CUDA_TRY(cudaMemcpyAsync(rows_out, h->mrows, (size_t)nrec * h->n_probe * S * 8, cudaMemcpyDeviceToHost,
                                     h->stream));
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    if (kernel_ms) cudaEventElapsedTime(kernel_ms, h->ev0, h->ev1);
    h->mcur = n_steps & 1;
    return 0;
}

// state of shot q after the last run (HOST concat of L_s*w per subdomain)
extern "C" int sfw_shots_state(sfw_stepper* h, int q, double* u_curr, double* u_prev) {
    char* errbuf = nullptr;
    int errlen = 0;
    if (!h->n_shots || q < 0 || q >= h->n_shots) return SFW_ECONFIG;
    const int S = h->n_shots;
    const long long total = (long long)h->n_sub * h->L * h->W;
    std::vector<double> buf((size_t)total * S);
    for (int lvl = 0; lvl < 2; ++lvl) {
        double* dst = lvl == 0 ? u_curr : u_prev;
        if (!dst) continue;
        const double* src = h->UM[lvl == 0 ? h->mcur : h->mcur ^ 1];
        SFW_CUDA_TRY(cudaMemcpy(buf.data(), src, buf.size() * 8, cudaMemcpyDeviceToHost));
        for (long long i = 0; i < total; ++i) dst[i] = buf[(size_t)i * S + q];
    }
    return 0;
}

// algorithmic bytes / flops per step of the multi-shot launch (SURVEY 8d, S shots)
extern "C" int sfw_shots_traffic(sfw_stepper* h, double* alg_bytes, double* alg_flops, double* streamed) {
    const double w = h->W, S = h->n_shots ? h->n_shots : 32;
    double b = 0, f = 0, s = 0;
    for (int i = 0; i < h->n_sub; ++i) {
        const double L = h->layers[i];
        b += 8.0 * ((2 * L - 1) * w * (w + 1) / 2 + 3 * L * w * S);
        f += S * (2.0 * (2 * L - 1) * w * w + 5 * L * w);
        s += 8.0 * (2 * L * h->TB + 3 * L * w * S);
    }
    if (alg_bytes) *alg_bytes = b;
    if (alg_flops) *alg_flops = f;
    if (streamed) *streamed = s;
    return 0;
}
