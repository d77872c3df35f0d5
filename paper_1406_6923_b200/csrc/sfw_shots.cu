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
    unsigned long long* dbg;  // debug cycle counters (SFW_MS_CLK builds) or null
    const double* mblk;       // [n_sub][6][M*M] interface mass per face (0 for outer faces)
    unsigned int* sflags;     // k_step_ms3: [n_sub][4] step tag of the published F_0 per shot group
    unsigned int tag0;        // k_step_ms3: tag of this launch's step 0 (monotone across launches)
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


// ---------------------------------------------------------------------------
// k_step_ms2: shot-column-parallel multi-shot stepping.  8 compute warps: warp
// (c, hh) owns shots 8c..8c+7 and output row tiles [hh*RH, hh*RH+RH) of every
// layer GEMM B X (B = Gamma_j or Gamma-hat_j, 56 x 56 symmetric, X 56 x 8), two
// warps per SMSP (the FP64 tensor pipe needs two LDS-fed DMMA streams per SMSP:
// measured 1 DMMA / 4.0 SM cycles with 8 warps vs 5.3 with 4).  Shots are
// independent: the two warps of a column pair exchange only their X rows
// (double-buffered, one 64-thread named barrier per GEMM); all warps share the
// TMA-streamed chain blocks and state blocks (full/empty mbarriers, 8 consumer
// arrivals per stage).  The lane's output fragment (row 8I + l/4, shots q0, q0+1)
// is also the slice of U / flux it owns in registers across the layer sweep.
//   per subdomain (A+B): F_0 = G_0 (U_1 - U_0) -> face buffer; acc_0 = H_0 F_0;
//     j = 1..L-1: F_j = G_j (U_{j+1} - U_j); A_j = H_j (F_j - F_{j-1}); leapfrog.
//   after all subdomains: step flag; neighbour flags; C: layer-1 coupling + leapfrog.
#ifndef SFW_M2_NC
#define SFW_M2_NC 4
#endif
#ifndef SFW_M2_SLEEP
#define SFW_M2_SLEEP 0
#endif
constexpr int M2_NC = SFW_M2_NC;  // chain-block stages
#if SFW_M2_SLEEP
#define M2_PWAIT mbar_wait_sleep
#else
#define M2_PWAIT mbar_wait
#endif
constexpr int M2_NSS = 8;   // state-block stages
#ifndef SFW_M2_SWZ
#define SFW_M2_SWZ 0
#endif
#if SFW_M2_SWZ
constexpr int M2_LDX = 8;   // X row stride; columns XOR-swizzled by m2_xs (conflict-free fragment reads)

// X / T tile element (row, col), col < 8: the column is XORed with 4 on row pairs 2,3 (mod 4), so
// the B-fragment reads (rows 4k+q, q < 4) and the double2 row writes are both bank-conflict free
__device__ __forceinline__ int m2_xs(int row, int col) { return row * M2_LDX + (col ^ (((row >> 1) & 1) << 2)); }
#else
constexpr int M2_LDX = 12;  // padded X row stride (conflict-free fragment reads)
__device__ __forceinline__ int m2_xs(int row, int col) { return row * M2_LDX + col; }
#endif
constexpr int M2_NQ = 4;    // warps per shot column tile (row-tile groups)
constexpr int M2_NW = 4 * M2_NQ;  // compute warps

template <int M, int HH>  // HH: row-tile group of this warp (0..M2_NQ-1)
__device__ __forceinline__ void ms2_compute(const MsParams& p, const double* cst, const double* sst, double* Xpair,
                                            uint64_t* cfull, uint64_t* cempty, uint64_t* sfull, uint64_t* sempty,
                                            uint64_t* stepdone, const int* ssub, const int* s_nb, int s0, int ns,
                                            int cw, int lane) {
    constexpr int S = 32;
    constexpr int RT = (6 * M + 7) / 8;
    constexpr int RH = (RT + M2_NQ - 1) / M2_NQ;  // row tiles per group
    constexpr int I0 = HH * RH;                   // first row tile of this warp
    constexpr int NI = (RT - I0 >= RH) ? RH : (RT - I0 > 0 ? RT - I0 : 1);  // row tiles of this warp (>= 1 slot)
    constexpr int WP = 8 * RT;
    constexpr int W = 6 * M;
    const int TB = p.TB, L = p.L;
    const long long K = p.K;
    const long long WS = (long long)W * S, KS = K * S;
    const int barP = 2 + cw;                    // named barrier of the column group (NQ warps)
    int tr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = 4 * h + (lane & 3), c = lane >> 2;
        tr[h] = (c >> 2) * 32 + r * 4 + (c & 3);
    }
    long long c_con = 0, s_con = 0;
    int xb = 0;  // X double buffer
#ifdef SFW_MS_CLK
    long long clk[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // c-wait, s-wait, gemm, total, flags, C, tail
    const long long clk_start = clock64();
#define MS_T0 const long long t0_ = clock64();
#define MS_T1(i) clk[i] += clock64() - t0_;
#else
#define MS_T0
#define MS_T1(i)
#endif
    auto c_acquire = [&]() -> const double* {
        const int st = (int)(c_con % M2_NC);
        MS_T0
        mbar_wait(&cfull[st], (uint32_t)((c_con / M2_NC) & 1));
        MS_T1(0)
        return cst + (size_t)st * TB;
    };
    auto c_release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty[c_con % M2_NC]);
        ++c_con;
    };
    auto s_acquire_at = [&](int o) -> const double* {  // o-th stage after the next unreleased one
        const long long c = s_con + o;
        const int st = (int)(c % M2_NSS);
        MS_T0
        mbar_wait(&sfull[st], (uint32_t)((c / M2_NSS) & 1));
        MS_T1(1)
        return sst + (size_t)st * WS;
    };
    auto s_release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[s_con % M2_NSS]);
        ++s_con;
    };
    const int r0 = lane >> 2;              // fragment row within a row tile
    const int q0 = 8 * cw + 2 * (lane & 3);  // first of the lane's two shots
    auto load_slice = [&](const double* blk, double (&v)[NI][2]) {
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int row = 8 * (I0 + i) + r0;
            if (row < W) {
                const double2 t = *reinterpret_cast<const double2*>(blk + (size_t)row * S + q0);
                v[i][0] = t.x;
                v[i][1] = t.y;
            } else {
                v[i][0] = v[i][1] = 0.0;
            }
        }
    };
    // write this warp's rows of X into the pair's next buffer, then meet the partner
    auto put_x = [&](const double (&v)[NI][2]) -> const double* {
        xb ^= 1;
        double* Xw = Xpair + (size_t)xb * WP * M2_LDX;
#pragma unroll
        for (int i = 0; i < NI; ++i)
            if (I0 + i < RT)
                *reinterpret_cast<double2*>(Xw + m2_xs(8 * (I0 + i) + r0, 2 * (lane & 3))) =
                    make_double2(v[i][0], v[i][1]);
        asm volatile("bar.sync %0, %1;" ::"r"(barP), "r"(M2_NQ * 32) : "memory");
        return Xw;
    };
    // acc = B X over this warp's row tiles, B symmetric (lower tiles, fragment order)
    // two accumulator chains per row tile (even / odd k-steps, summed at the end): 2 NI independent
    // DMMA chains per warp, so one warp alone keeps its SMSP's FP64 tensor pipe fed
    auto gemm = [&](const double* tiles, const double* Xw, double (&acc)[NI][2]) {
        MS_T0
        double acc2[NI][2];
#pragma unroll
        for (int i = 0; i < NI; ++i) acc[i][0] = acc[i][1] = acc2[i][0] = acc2[i][1] = 0.0;
#pragma unroll
        for (int kap = 0; kap < 2 * RT; ++kap) {
            const int Kt = kap >> 1, h = kap & 1;
            const double b = Xw[m2_xs(4 * kap + (lane & 3), r0)];
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int I = I0 + i;
                if (I >= RT) break;
                const double a = (I >= Kt) ? tiles[(I * (I + 1) / 2 + Kt) * 64 + h * 32 + lane]
                                           : tiles[(Kt * (Kt + 1) / 2 + I) * 64 + tr[h]];
                if (h)
                    dmma8x8x4(acc2[i], a, b);
                else
                    dmma8x8x4(acc[i], a, b);
            }
        }
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            acc[i][0] += acc2[i][0];
            acc[i][1] += acc2[i][1];
        }
#ifdef SFW_MS_CLK
        for (int i = 0; i < NI; ++i) asm volatile("" ::"d"(acc[i][0]), "d"(acc[i][1]));
#endif
        MS_T1(2)
    };
    auto store_global = [&](double* blk, const double (&v)[NI][2]) {
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int row = 8 * (I0 + i) + r0;
            if (row < W) *reinterpret_cast<double2*>(blk + (size_t)row * S + q0) = make_double2(v[i][0], v[i][1]);
        }
    };
    const double dt2 = p.dt2;
    const bool src0 = ssub[q0] >= 0, src1 = ssub[q0 + 1] >= 0;

#ifndef SFW_M2_LAG
#define SFW_M2_LAG 0
#endif
#ifdef SFW_M2_FAKE_STATE  // timing experiment: state reads all hit the CTA's first subdomain (L2)
#define M2_FAKE_S 1
#else
#define M2_FAKE_S 0
#endif
    for (int k = 1; k <= p.n_steps; ++k) {
        const int par = k & 1;
        const int cb = (k - 1) & 1;
        double* Un = cb ? p.U0 : p.U1;
        double* fx = p.flux + (size_t)par * p.n_sub * WS;
        const int kk = k - 1;
        const double f0 = src0 ? p.ftab[(size_t)q0 * p.ftab_stride + kk] : 0.0;
        const double f1 = src1 ? p.ftab[(size_t)(q0 + 1) * p.ftab_stride + kk] : 0.0;
        double sq0 = 0.0, sq1 = 0.0;
        if (SFW_M2_LAG > 0 && cw >= 2) __nanosleep(SFW_M2_LAG);  // column groups 2,3 trail 0,1
        auto force = [&](int s, long long idx, int e) -> double {  // shot source term (ssub[q] == s)
            const int q = q0 + e;
            return __dmul_rn(p.shot_vec[p.shot_voff[q] + idx], e ? f1 : f0);
        };

        // ---------------- A + B: every subdomain's layer sweep --------------------------
        for (int sl = 0; sl < ns; ++sl) {
            const int s = s0 + sl;
            double ua[NI][2], ub[NI][2], fp[NI][2], acc[NI][2];
            const double* Xw;
            {
                double u0[NI][2];
                load_slice(s_acquire_at(0), u0);
                load_slice(s_acquire_at(1), ua);  // U_1
                s_release();
                s_release();
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    u0[i][0] = ua[i][0] - u0[i][0];
                    u0[i][1] = ua[i][1] - u0[i][1];
                }
                Xw = put_x(u0);
            }
            gemm(c_acquire(), Xw, fp);  // F_0
            c_release();
            store_global(fx + (size_t)s * WS, fp);
            const bool interior = s_nb[sl * 6] >= 0 && s_nb[sl * 6 + 1] >= 0 && s_nb[sl * 6 + 2] >= 0 &&
                                  s_nb[sl * 6 + 3] >= 0 && s_nb[sl * 6 + 4] >= 0 && s_nb[sl * 6 + 5] >= 0;
            if (!interior) {  // acc_0 = H_0 F_0: only outer-face rows are ever read back
                Xw = put_x(fp);
                gemm(c_acquire(), Xw, acc);
                c_release();
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int row = 8 * (I0 + i) + r0;
                    if (row < W && s_nb[sl * 6 + row / M] < 0)
                        *reinterpret_cast<double2*>(p.acc1 + ((size_t)s * W + row) * S + q0) =
                            make_double2(acc[i][0], acc[i][1]);
                }
            }
            for (int j = 1; j < L; ++j) {
                if (j + 1 < L) {
                    load_slice(s_acquire_at(0), ub);  // U_{j+1}
                    s_release();
                } else {
#pragma unroll
                    for (int i = 0; i < NI; ++i) ub[i][0] = ub[i][1] = 0.0;
                }
                {
                    double x[NI][2];
#pragma unroll
                    for (int i = 0; i < NI; ++i) {
                        x[i][0] = ub[i][0] - ua[i][0];
                        x[i][1] = ub[i][1] - ua[i][1];
                    }
                    Xw = put_x(x);
                }
                gemm(c_acquire(), Xw, acc);  // F_j
                c_release();
                {
                    double x[NI][2];
#pragma unroll
                    for (int i = 0; i < NI; ++i) {
                        x[i][0] = acc[i][0] - fp[i][0];
                        x[i][1] = acc[i][1] - fp[i][1];
                        fp[i][0] = acc[i][0];
                        fp[i][1] = acc[i][1];
                    }
                    Xw = put_x(x);
                }
                double uo[NI][2];
                load_slice(s_acquire_at(0), uo);  // Uprev_j
                s_release();
                gemm(c_acquire(), Xw, acc);  // A_j
                c_release();
                double* un = Un + (size_t)s * KS + (size_t)j * WS;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int row = 8 * (I0 + i) + r0;
                    double v[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        double tot = acc[i][e];
                        if ((e ? src1 : src0) && row < W && ssub[q0 + e] == s)
                            tot = __dadd_rn(tot, force(s, (long long)j * W + row, e));
                        v[e] = __dadd_rn(__dsub_rn(__dmul_rn(2.0, ua[i][e]), uo[i][e]), __dmul_rn(dt2, tot));
                    }
                    if (row < W) {
                        *reinterpret_cast<double2*>(un + (size_t)row * S + q0) = make_double2(v[0], v[1]);
                        sq0 = fma(v[0], v[0], sq0);
                        sq1 = fma(v[1], v[1], sq1);
                    }
                }
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    ua[i][0] = ub[i][0];
                    ua[i][1] = ub[i][1];
                }
            }
        }
        // ---------------- step flag, neighbour flags ------------------------------------
#ifdef SFW_MS_CLK
        long long tf0 = clock64();
#endif
        asm volatile("bar.sync 1, %0;" ::"r"(M2_NW * 32) : "memory");
        if (cw == 0 && HH == 0 && lane == 0) flag_publish(p.flags, (unsigned int)k);
        if (cw == 0 && HH == 0)
            flags_wait(p.flags, p.ncta + p.ncta_ptr[blockIdx.x], p.ncta_ptr[blockIdx.x + 1] - p.ncta_ptr[blockIdx.x],
                       (unsigned int)k, lane);
        asm volatile("bar.sync 1, %0;" ::"r"(M2_NW * 32) : "memory");
#ifdef SFW_MS_CLK
        clk[4] += clock64() - tf0;
        tf0 = clock64();
#endif
        // ---------------- C: layer-1 face coupling + leapfrog ---------------------------
        for (int sl = 0; sl < ns; ++sl) {
            const int s = s0 + sl;
            const double* mb = s_acquire_at(0);  // [6][M][M] interface mass
            // own + neighbour layer-1 flux of every face row, the pair's 8 shots; each warp
            // of the pair stages half of the rows (independent loads: one L2 round trip)
            xb ^= 1;
            double* T = Xpair + (size_t)xb * WP * M2_LDX;
            {
                constexpr int NROW = (6 * M + M2_NQ - 1) / M2_NQ;  // rows per warp
                constexpr int NIT = (NROW * 4 + 31) / 32;
                double2 ow[NIT], ot[NIT];
#pragma unroll
                for (int t = 0; t < NIT; ++t) {
                    const int it = lane + 32 * t, row = HH * NROW + (it >> 2), pr = it & 3;
                    ow[t] = ot[t] = make_double2(0.0, 0.0);
                    if ((it >> 2) < NROW && row < 6 * M) {
                        const int f = row / M, c = row % M, nb = s_nb[sl * 6 + f];
                        if (nb >= 0) {
                            ow[t] = __ldcg(reinterpret_cast<const double2*>(fx + ((size_t)s * W + row) * S + 8 * cw + 2 * pr));
                            ot[t] = __ldcg(reinterpret_cast<const double2*>(fx + ((size_t)nb * W + (f ^ 1) * M + c) * S +
                                                                           8 * cw + 2 * pr));
                        }
                    }
                }
#pragma unroll
                for (int t = 0; t < NIT; ++t) {
                    const int it = lane + 32 * t, row = HH * NROW + (it >> 2), pr = it & 3;
                    if ((it >> 2) < NROW && row < 6 * M)
                        *reinterpret_cast<double2*>(T + m2_xs(row, 2 * pr)) =
                            make_double2(__dadd_rn(ow[t].x, ot[t].x), __dadd_rn(ow[t].y, ot[t].y));
                }
            }
            double a1[NI][2];
#pragma unroll
            for (int i = 0; i < NI; ++i) {  // boundary-face accelerations (prefetch)
                const int row = 8 * (I0 + i) + r0;
                a1[i][0] = a1[i][1] = 0.0;
                if (row < W && s_nb[sl * 6 + row / M] < 0) {
                    const double2 t = __ldcg(reinterpret_cast<const double2*>(p.acc1 + ((size_t)s * W + row) * S + q0));
                    a1[i][0] = t.x;
                    a1[i][1] = t.y;
                }
            }
            asm volatile("bar.sync %0, %1;" ::"r"(barP), "r"(M2_NQ * 32) : "memory");
            double u0[NI][2], uo[NI][2];
            load_slice(s_acquire_at(1), u0);
            load_slice(s_acquire_at(2), uo);
            double* un = Un + (size_t)s * KS;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int row = 8 * (I0 + i) + r0;
                if (row >= W) continue;
                const int f = row / M, r = row % M;
                double a[2] = {a1[i][0], a1[i][1]};
                if (s_nb[sl * 6 + f] >= 0) {
                    a[0] = a[1] = 0.0;
                    const double* mx = mb + (f * M + r) * M;
#pragma unroll
                    for (int c = 0; c < M; ++c) {
                        const double mc = mx[c];
                        const double2 t = *reinterpret_cast<const double2*>(T + m2_xs(f * M + c, 2 * (lane & 3)));
                        a[0] = fma(mc, t.x, a[0]);
                        a[1] = fma(mc, t.y, a[1]);
                    }
                }
                double v[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    double tot = a[e];
                    if ((e ? src1 : src0) && ssub[q0 + e] == s) tot = __dadd_rn(tot, force(s, row, e));
                    v[e] = __dadd_rn(__dsub_rn(__dmul_rn(2.0, u0[i][e]), uo[i][e]), __dmul_rn(dt2, tot));
                }
                *reinterpret_cast<double2*>(un + (size_t)row * S + q0) = make_double2(v[0], v[1]);
                sq0 = fma(v[0], v[0], sq0);
                sq1 = fma(v[1], v[1], sq1);
            }
            s_release();  // mass
            s_release();  // U_0
            s_release();  // Uprev_0
        }
#ifdef SFW_MS_CLK
        clk[5] += clock64() - tf0;
        tf0 = clock64();
#endif
        // per-shot |U|^2 of this warp's rows: lanes with equal (lane & 3) hold the same shots;
        // the pair's two halves go to separate partial slots (k_ms_norms sums them)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            sq0 += __shfl_xor_sync(0xffffffffu, sq0, o);
            sq1 += __shfl_xor_sync(0xffffffffu, sq1, o);
        }
        if (lane < 4) {
            double* np = p.norm_part + (((size_t)kk * gridDim.x + blockIdx.x) * M2_NQ + HH) * S + q0;
            np[0] = sq0;
            np[1] = sq1;
        }
        // probes (this warp: its pair's 8 shots, every other probe): rows of U after the step
        if (k % p.record_every == 0 && p.rows) {
            asm volatile("bar.sync %0, %1;" ::"r"(barP), "r"(M2_NQ * 32) : "memory");  // group's U rows written
            const long long row = k / p.record_every - 1;
            const int q = 8 * cw + (lane & 7);
            for (int s = s0; s < s0 + ns; ++s) {
                const double* us = Un + (size_t)s * KS;
                for (int pq = p.prb_ptr[s] + M2_NQ * (lane >> 3) + HH; pq < p.prb_ptr[s + 1]; pq += 4 * M2_NQ) {
                    const int pid = p.prb_ids[pq];
                    const int tap = p.prb_tap[pid];
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
        // this step's state writes feed the next step's TMA reads (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(stepdone);
#ifdef SFW_MS_CLK
        clk[6] += clock64() - tf0;
#endif
    }
#ifdef SFW_MS_CLK
    clk[3] = clock64() - clk_start;
    if (lane < 8 && p.dbg) {
        long long v = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (lane == i) v = clk[i];
        p.dbg[(blockIdx.x * M2_NW + M2_NQ * cw + HH) * 8 + lane] = v;
    }
#endif
#undef MS_T0
#undef MS_T1
}

template <int M>
__global__ void __launch_bounds__((M2_NW + 2) * 32, 1) k_step_ms2(const MsParams p) {
    constexpr int S = 32;
    constexpr int RT = (6 * M + 7) / 8;
    constexpr int WP = 8 * RT;
    constexpr int W = 6 * M;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = p.L, TB = p.TB;
    const long long K = p.K;
    const long long WS = (long long)W * S, KS = K * S;
    double* cst = reinterpret_cast<double*>(smem_raw);   // [NC][TB]
    double* sst = cst + (size_t)M2_NC * TB;              // [NSS][W*S]
    double* Xall = sst + (size_t)M2_NSS * WS;            // [4 column groups][2][WP][LDX]
    uint64_t* cfull = reinterpret_cast<uint64_t*>(Xall + (size_t)4 * 2 * WP * M2_LDX);
    uint64_t* cempty = cfull + M2_NC;
    uint64_t* sfull = cempty + M2_NC;
    uint64_t* sempty = sfull + M2_NSS;
    uint64_t* stepdone = sempty + M2_NSS;
    int* ssub = reinterpret_cast<int*>(stepdone + 1);
    int* s_nb = ssub + S;  // [ns][6] face neighbours of the CTA's subdomains

    for (int q = threadIdx.x; q < S; q += blockDim.x) ssub[q] = p.shot_sub[q];
    if (threadIdx.x == 0) {
        for (int i = 0; i < M2_NC; ++i) {
            mbar_init(&cfull[i], 1);
            mbar_init(&cempty[i], M2_NW);
        }
        for (int i = 0; i < M2_NSS; ++i) {
            mbar_init(&sfull[i], 1);
            mbar_init(&sempty[i], M2_NW);
        }
        mbar_init(stepdone, M2_NW);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 4 * 2 * WP * M2_LDX; i += blockDim.x) Xall[i] = 0.0;
    const int s0 = p.cta_sub_ptr[blockIdx.x], s1 = p.cta_sub_ptr[blockIdx.x + 1];
    const int ns = s1 - s0;
    for (int i = threadIdx.x; i < ns * 6; i += blockDim.x) s_nb[i] = p.nbr[s0 * 6 + i];
    __syncthreads();

    // ======== producer warps: chain blocks (ungated) and state blocks (gated per step) ====
    // one warp per ring (lane 0 issues); waits are blocking mbarrier try_waits, so the producers
    // take no issue slots from the compute warps while their ring is full.  Interior subdomains
    // never read acc_0 (only outer-face rows do), so their Gamma-hat_0 block is not streamed.
    if (warp >= M2_NW) {
        if (lane == 0 && warp == M2_NW) {  // chain-block ring
            const uint64_t pol = l2_policy_evict_first();
            const uint32_t cbytes = (uint32_t)TB * 8u;
            long long c_iss = 0;
            for (int k = 0; k < p.n_steps; ++k)
                for (int sl = 0; sl < ns; ++sl) {
                    const bool interior = s_nb[sl * 6] >= 0 && s_nb[sl * 6 + 1] >= 0 && s_nb[sl * 6 + 2] >= 0 &&
                                          s_nb[sl * 6 + 3] >= 0 && s_nb[sl * 6 + 4] >= 0 && s_nb[sl * 6 + 5] >= 0;
                    for (int b = 0; b < 2 * L; ++b) {
                        if (b == 1 && interior) continue;
                        const int st = (int)(c_iss % M2_NC);
                        M2_PWAIT(&cempty[st], (uint32_t)(((c_iss / M2_NC) & 1) ^ 1));
                        mbar_arrive_expect_tx(&cfull[st], cbytes);
#ifdef SFW_M2_FAKE_CHAIN  // timing experiment: every CTA streams its first subdomain's blocks (L2 hits)
                        bulk_g2s(cst + (size_t)st * TB, p.tcoef + ((long long)(s0) * 2 * L + b) * TB, cbytes,
                                 &cfull[st], pol);
#else
                        bulk_g2s(cst + (size_t)st * TB, p.tcoef + ((long long)(s0 + sl) * 2 * L + b) * TB, cbytes,
                                 &cfull[st], pol);
#endif
                        ++c_iss;
                    }
                }
        } else if (lane == 0 && warp == M2_NW + 1) {  // state-block ring, gated per step
            const uint64_t pol_state = l2_policy_evict_first();  // measured 1-1.5% faster than evict_last
            const uint32_t mbytes = (uint32_t)(6 * M * M * 8);
            const uint32_t sbytes = (uint32_t)(WS * 8);
            const int nab = 2 * L - 1;
            long long s_iss = 0;
            for (int k = 0; k < p.n_steps; ++k) {
                // step k >= 1 reads what step k-1 wrote: wait for all compute warps
                if (k > 0) M2_PWAIT(stepdone, (uint32_t)((k - 1) & 1));
                const int cb = k & 1;
                const double* cur = cb ? p.U1 : p.U0;
                const double* prv = cb ? p.U0 : p.U1;
                for (int spos = 0; spos < ns * (nab + 3); ++spos) {
                    const double* src;
                    uint32_t bytes = sbytes;
                    if (spos < ns * nab) {
                        const int sl = M2_FAKE_S ? 0 : spos / nab, r = spos % nab;
                        const long long base = (long long)(s0 + sl) * KS;
                        if (r < 2) {
                            src = cur + base + r * WS;  // U_0, U_1
                        } else {
                            const int rp = r - 2;  // j = 1..L-1: [U_{j+1}], Uprev_j
                            if (rp < 2 * (L - 2)) {
                                const int j = 1 + rp / 2;
                                src = (rp & 1) ? prv + base + j * WS : cur + base + (j + 1) * WS;
                            } else {
                                src = prv + base + (L - 1) * WS;
                            }
                        }
                    } else {
                        const int r = spos - ns * nab, sl = M2_FAKE_S ? 0 : r / 3, w3 = r % 3;
                        if (w3 == 0) {  // interface mass of the 6 faces
                            src = p.mblk + (size_t)(s0 + sl) * 6 * M * M;
                            bytes = mbytes;
                        } else {
                            src = ((w3 == 2) ? prv : cur) + (long long)(s0 + sl) * KS;  // U_0, Uprev_0
                        }
                    }
                    const int st = (int)(s_iss % M2_NSS);
                    M2_PWAIT(&sempty[st], (uint32_t)(((s_iss / M2_NSS) & 1) ^ 1));
                    mbar_arrive_expect_tx(&sfull[st], bytes);
                    bulk_g2s(sst + (size_t)st * WS, src, bytes, &sfull[st], pol_state);
                    ++s_iss;
                }
            }
        }
        return;
    }
    // ======== compute warps: (column tile cw, row half hh) ========
    // SMSP (warp % 4) hosts one warp of every row-tile group -> equal DMMA work per SMSP
    const int cw = warp / M2_NQ, hh = (warp / M2_NQ + warp) % M2_NQ;
    double* Xpair = Xall + (size_t)cw * 2 * WP * M2_LDX;
    switch (hh) {
        case 0: ms2_compute<M, 0>(p, cst, sst, Xpair, cfull, cempty, sfull, sempty, stepdone, ssub, s_nb, s0, ns, cw, lane); break;
        case 1: ms2_compute<M, 1>(p, cst, sst, Xpair, cfull, cempty, sfull, sempty, stepdone, ssub, s_nb, s0, ns, cw, lane); break;
        case 2: ms2_compute<M, 2>(p, cst, sst, Xpair, cfull, cempty, sfull, sempty, stepdone, ssub, s_nb, s0, ns, cw, lane); break;
        default: ms2_compute<M, 3>(p, cst, sst, Xpair, cfull, cempty, sfull, sempty, stepdone, ssub, s_nb, s0, ns, cw, lane); break;
    }
}

static size_t ms2_smem_bytes(int RT, int TB, int W, int nsmax) {
    return 8 * ((size_t)M2_NC * TB + (size_t)M2_NSS * W * 32 + (size_t)4 * 2 * 8 * RT * M2_LDX + 2 * M2_NC +
                2 * M2_NSS + 1) +
           4 * (32 + 6 * (size_t)nsmax) + 64;
}

// ---------------------------------------------------------------------------
// k_step_ms4: two-team multi-shot stepping (config 4 default).
//
// k_step_ms2 splits every GEMM's output rows over the 4 warps of a shot column, so each of the
// 17-18 GEMMs of a subdomain sweep ends in a named barrier (X exchange) and every warp reaches its
// ring waits and barriers at the same time as all others: measured, feeding every chain and state
// block from L2 did not change its step time at all (0.760 ms both ways) -- the DMMA pipe idles in
// the synchronised non-GEMM stretches, not for lack of bytes.
//
// Here a warp owns 8 shots and ALL row tiles of its GEMMs (Y = B X, 56 x 8 per warp, 7 row tiles x
// 14 k-steps = 98 DMMA), so the layer sweep needs no cross-warp exchange: X goes through a per-warp
// shared-memory tile (__syncwarp only).  The 8 compute warps form two teams of 4 (one warp per
// 8-shot column); team t sweeps subdomains sl = t, t+2, ... of the CTA with its own chain-block
// and state-block rings and its own producer warps, so the teams drift independently and one
// team's non-GEMM work (ring waits, X transposes, leapfrog, stores) overlaps the other team's
// DMMA on the same SMSP (each SMSP hosts one warp of each team and one producer warp).
// Per subdomain the arithmetic is that of k_step_ms2 (stepper.py:243-389 per shot):
//   F_0 = G_0 (U_1 - U_0) -> face buffer;  acc_0 = H_0 F_0 (outer faces only);
//   j = 1..L-1: F_j = G_j (U_{j+1} - U_j); A_j = H_j (F_j - F_{j-1}); leapfrog of layer j;
// then, after the CTA's step flag and its neighbours' (phase C): layer-0 face coupling
// mass (own + neighbour F_0) and leapfrog, per-shot |U|^2 partials, probe rows.
constexpr int M4_NC = 3;     // chain-block stages per team
constexpr int M4_NSS = 3;    // state-block stages per team
constexpr int M4_LDX = 12;   // X row stride (conflict-free fragment reads)
constexpr int M4_NT = 2;     // teams
constexpr int M4_NW = 4 * M4_NT;  // compute warps

template <int M>
__device__ __forceinline__ void ms4_compute(const MsParams& p, const double* cst, const double* sst, double* Xs,
                                            uint64_t* cfull, uint64_t* cempty, uint64_t* sfull, uint64_t* sempty,
                                            uint64_t* stepdone, const int* ssub, const int* s_nb, int s0, int ns,
                                            int team, int cw, int lane) {
    constexpr int S = 32;
    constexpr int RT = (6 * M + 7) / 8;
    constexpr int W = 6 * M;
    const int TB = p.TB, L = p.L;
    const long long K = p.K;
    const long long WS = (long long)W * S, KS = K * S;
    int tr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = 4 * h + (lane & 3), c = lane >> 2;
        tr[h] = (c >> 2) * 32 + r * 4 + (c & 3);
    }
    long long c_con = 0, s_con = 0;
#ifdef SFW_MS_CLK
    long long clk[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // c-wait, s-wait, gemm, total, flags, C, -, -
    const long long clk_start = clock64();
#define M4_T0 const long long t0_ = clock64();
#define M4_T1(i) clk[i] += clock64() - t0_;
#else
#define M4_T0
#define M4_T1(i)
#endif
    auto c_acquire = [&]() -> const double* {
        const int st = (int)(c_con % M4_NC);
        M4_T0
        mbar_wait(&cfull[st], (uint32_t)((c_con / M4_NC) & 1));
        M4_T1(0)
        return cst + (size_t)st * TB;
    };
    auto c_release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty[c_con % M4_NC]);
        ++c_con;
    };
    auto s_acquire = [&]() -> const double* {
        const int st = (int)(s_con % M4_NSS);
        M4_T0
        mbar_wait(&sfull[st], (uint32_t)((s_con / M4_NSS) & 1));
        M4_T1(1)
        return sst + (size_t)st * WS;
    };
    auto s_release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[s_con % M4_NSS]);
        ++s_con;
    };
    const int r0 = lane >> 2;                 // fragment row within a row tile
    const int q0 = 8 * cw + 2 * (lane & 3);   // first of the lane's two shots
    // the lane's slice of a W x S block: rows 8I + r0 (I < RT), shots q0, q0 + 1
    auto load_slice = [&](const double* blk, double (&v)[RT][2]) {
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            const int row = 8 * i + r0;
            if (row < W) {
                const double2 t = *reinterpret_cast<const double2*>(blk + (size_t)row * S + q0);
                v[i][0] = t.x;
                v[i][1] = t.y;
            } else {
                v[i][0] = v[i][1] = 0.0;
            }
        }
    };
    auto store_global = [&](double* blk, const double (&v)[RT][2]) {
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            const int row = 8 * i + r0;
            if (row < W) *reinterpret_cast<double2*>(blk + (size_t)row * S + q0) = make_double2(v[i][0], v[i][1]);
        }
    };
    // X (56 x 8, this warp's shots) into the warp's own tile; padding rows carry zeros
    auto put_x = [&](const double (&v)[RT][2]) {
        __syncwarp();  // previous GEMM's reads of Xs are done
#pragma unroll
        for (int i = 0; i < RT; ++i)
            *reinterpret_cast<double2*>(Xs + (8 * i + r0) * M4_LDX + 2 * (lane & 3)) = make_double2(v[i][0], v[i][1]);
        __syncwarp();
    };
    // acc = B X, B symmetric (lower 8x8 tiles in DMMA fragment order), all RT row tiles
    auto gemm = [&](const double* tiles, double (&acc)[RT][2]) {
        M4_T0
#pragma unroll
        for (int i = 0; i < RT; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
        for (int kap = 0; kap < 2 * RT; ++kap) {
            const int Kt = kap >> 1, h = kap & 1;
            const double b = Xs[(4 * kap + (lane & 3)) * M4_LDX + r0];
#pragma unroll
            for (int I = 0; I < RT; ++I) {
                const double a = (I >= Kt) ? tiles[(I * (I + 1) / 2 + Kt) * 64 + h * 32 + lane]
                                           : tiles[(Kt * (Kt + 1) / 2 + I) * 64 + tr[h]];
                dmma8x8x4(acc[I], a, b);
            }
        }
#ifdef SFW_MS_CLK
        for (int i = 0; i < RT; ++i) asm volatile("" ::"d"(acc[i][0]), "d"(acc[i][1]));
#endif
        M4_T1(2)
    };
    const double dt2 = p.dt2;
    const bool src0 = ssub[q0] >= 0, src1 = ssub[q0 + 1] >= 0;
    auto interior_of = [&](int sl) {
        return s_nb[sl * 6] >= 0 && s_nb[sl * 6 + 1] >= 0 && s_nb[sl * 6 + 2] >= 0 && s_nb[sl * 6 + 3] >= 0 &&
               s_nb[sl * 6 + 4] >= 0 && s_nb[sl * 6 + 5] >= 0;
    };

    for (int k = 1; k <= p.n_steps; ++k) {
        const int par = k & 1;
        const int cb = (k - 1) & 1;
        double* Un = cb ? p.U0 : p.U1;
        double* fx = p.flux + (size_t)par * p.n_sub * WS;
        const int kk = k - 1;
        const double f0 = src0 ? p.ftab[(size_t)q0 * p.ftab_stride + kk] : 0.0;
        const double f1 = src1 ? p.ftab[(size_t)(q0 + 1) * p.ftab_stride + kk] : 0.0;
        double sq0 = 0.0, sq1 = 0.0;
        auto force = [&](long long idx, int e) -> double {  // shot source term (ssub[q] == s)
            return __dmul_rn(p.shot_vec[p.shot_voff[q0 + e] + idx], e ? f1 : f0);
        };

        // ---------------- A: layer-0 fluxes of this team's subdomains ----------------------
        for (int sl = team; sl < ns; sl += M4_NT) {
            const int s = s0 + sl;
            double ua[RT][2], fp[RT][2], x[RT][2];
            load_slice(s_acquire(), x);  // U_0
            s_release();
            load_slice(s_acquire(), ua);  // U_1
            s_release();
#pragma unroll
            for (int i = 0; i < RT; ++i) {
                x[i][0] = ua[i][0] - x[i][0];
                x[i][1] = ua[i][1] - x[i][1];
            }
            put_x(x);
            gemm(c_acquire(), fp);  // F_0
            c_release();
            store_global(fx + (size_t)s * WS, fp);
            if (!interior_of(sl)) {  // acc_0 = H_0 F_0: only outer-face rows are ever read back
                put_x(fp);
                gemm(c_acquire(), x);
                c_release();
#pragma unroll
                for (int i = 0; i < RT; ++i) {
                    const int row = 8 * i + r0;
                    if (row < W && s_nb[sl * 6 + row / M] < 0)
                        *reinterpret_cast<double2*>(p.acc1 + ((size_t)s * W + row) * S + q0) =
                            make_double2(x[i][0], x[i][1]);
                }
            }
        }
        // ---------------- step flag after phase A, neighbour flags (both teams) --------------
#ifdef SFW_MS_CLK
        long long tf0 = clock64();
#endif
        asm volatile("bar.sync 1, %0;" ::"r"(M4_NW * 32) : "memory");
        if (team == 0 && cw == 0 && lane == 0) flag_publish(p.flags, (unsigned int)k);
        if (team == 0 && cw == 0)
            flags_wait(p.flags, p.ncta + p.ncta_ptr[blockIdx.x], p.ncta_ptr[blockIdx.x + 1] - p.ncta_ptr[blockIdx.x],
                       (unsigned int)k, lane);
        asm volatile("bar.sync 1, %0;" ::"r"(M4_NW * 32) : "memory");
#ifdef SFW_MS_CLK
        clk[4] += clock64() - tf0;
#endif
        // ---------------- per subdomain: C (layer-0 coupling + leapfrog), then B (layers >= 1)
        for (int sl = team; sl < ns; sl += M4_NT) {
            const int s = s0 + sl;
#ifdef SFW_MS_CLK
            long long tc0 = clock64();
#endif
            {
                double u0[RT][2], uo[RT][2];
                load_slice(s_acquire(), u0);  // U_0
                s_release();
                load_slice(s_acquire(), uo);  // Uprev_0
                s_release();
                const double* mb = s_acquire();  // [6][M][M] interface mass
                // own + neighbour F_0 of every shared-face row, this warp's 8 shots, into its tile
                __syncwarp();
                constexpr int NIT = (W * 4 + 31) / 32;
                double2 ow[NIT], ot[NIT];
#pragma unroll
                for (int t = 0; t < NIT; ++t) {  // all loads first (one L2 round trip)
                    const int it = lane + 32 * t, row = it >> 2, pr = it & 3;
                    ow[t] = ot[t] = make_double2(0.0, 0.0);
                    if (row < W) {
                        const int f = row / M, c = row % M, nb = s_nb[sl * 6 + f];
                        if (nb >= 0) {
                            ow[t] = __ldcg(reinterpret_cast<const double2*>(fx + ((size_t)s * W + row) * S + 8 * cw +
                                                                            2 * pr));
                            ot[t] = __ldcg(reinterpret_cast<const double2*>(
                                fx + ((size_t)nb * W + (f ^ 1) * M + c) * S + 8 * cw + 2 * pr));
                        }
                    }
                }
                double a1[RT][2];
#pragma unroll
                for (int i = 0; i < RT; ++i) {  // outer-face accelerations
                    const int row = 8 * i + r0;
                    a1[i][0] = a1[i][1] = 0.0;
                    if (row < W && s_nb[sl * 6 + row / M] < 0) {
                        const double2 t = __ldcg(reinterpret_cast<const double2*>(p.acc1 + ((size_t)s * W + row) * S + q0));
                        a1[i][0] = t.x;
                        a1[i][1] = t.y;
                    }
                }
#pragma unroll
                for (int t = 0; t < NIT; ++t) {
                    const int it = lane + 32 * t, row = it >> 2, pr = it & 3;
                    if (row < W)
                        *reinterpret_cast<double2*>(Xs + row * M4_LDX + 2 * pr) =
                            make_double2(__dadd_rn(ow[t].x, ot[t].x), __dadd_rn(ow[t].y, ot[t].y));
                }
                __syncwarp();
                double* un = Un + (size_t)s * KS;
#pragma unroll
                for (int i = 0; i < RT; ++i) {
                    const int row = 8 * i + r0;
                    if (row >= W) continue;
                    const int f = row / M, r = row % M;
                    double a[2] = {a1[i][0], a1[i][1]};
                    if (s_nb[sl * 6 + f] >= 0) {
                        a[0] = a[1] = 0.0;
                        const double* mx = mb + (f * M + r) * M;
#pragma unroll
                        for (int c = 0; c < M; ++c) {
                            const double mc = mx[c];
                            const double2 t = *reinterpret_cast<const double2*>(Xs + (f * M + c) * M4_LDX + 2 * (lane & 3));
                            a[0] = fma(mc, t.x, a[0]);
                            a[1] = fma(mc, t.y, a[1]);
                        }
                    }
                    double v[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        double tot = a[e];
                        if ((e ? src1 : src0) && ssub[q0 + e] == s) tot = __dadd_rn(tot, force(row, e));
                        v[e] = __dadd_rn(__dsub_rn(__dmul_rn(2.0, u0[i][e]), uo[i][e]), __dmul_rn(dt2, tot));
                    }
                    *reinterpret_cast<double2*>(un + (size_t)row * S + q0) = make_double2(v[0], v[1]);
                    sq0 = fma(v[0], v[0], sq0);
                    sq1 = fma(v[1], v[1], sq1);
                }
                s_release();  // mass
            }
#ifdef SFW_MS_CLK
            clk[5] += clock64() - tc0;
#endif
            // B: layers 1..L-1 (F_0 of this warp's rows and shots re-read from the face buffer)
            double ua[RT][2], fp[RT][2], acc[RT][2];
            load_slice(s_acquire(), ua);  // U_1
            s_release();
#pragma unroll
            for (int i = 0; i < RT; ++i) {
                const int row = 8 * i + r0;
                fp[i][0] = fp[i][1] = 0.0;
                if (row < W) {
                    const double2 t = *reinterpret_cast<const double2*>(fx + ((size_t)s * W + row) * S + q0);
                    fp[i][0] = t.x;
                    fp[i][1] = t.y;
                }
            }
            for (int j = 1; j < L; ++j) {
                double x[RT][2];
                if (j + 1 < L) {
                    load_slice(s_acquire(), x);  // U_{j+1}
                    s_release();
                } else {
#pragma unroll
                    for (int i = 0; i < RT; ++i) x[i][0] = x[i][1] = 0.0;
                }
                double d[RT][2];
#pragma unroll
                for (int i = 0; i < RT; ++i) {
                    d[i][0] = x[i][0] - ua[i][0];
                    d[i][1] = x[i][1] - ua[i][1];
                }
                put_x(d);
                gemm(c_acquire(), acc);  // F_j
                c_release();
#pragma unroll
                for (int i = 0; i < RT; ++i) {
                    d[i][0] = acc[i][0] - fp[i][0];
                    d[i][1] = acc[i][1] - fp[i][1];
                    fp[i][0] = acc[i][0];
                    fp[i][1] = acc[i][1];
                }
                put_x(d);
                gemm(c_acquire(), acc);  // A_j
                c_release();
                double uo[RT][2];
                load_slice(s_acquire(), uo);  // Uprev_j
                s_release();
                double* un = Un + (size_t)s * KS + (size_t)j * WS;
#pragma unroll
                for (int i = 0; i < RT; ++i) {
                    const int row = 8 * i + r0;
                    double v[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        double tot = acc[i][e];
                        if ((e ? src1 : src0) && row < W && ssub[q0 + e] == s)
                            tot = __dadd_rn(tot, force((long long)j * W + row, e));
                        v[e] = __dadd_rn(__dsub_rn(__dmul_rn(2.0, ua[i][e]), uo[i][e]), __dmul_rn(dt2, tot));
                    }
                    if (row < W) {
                        *reinterpret_cast<double2*>(un + (size_t)row * S + q0) = make_double2(v[0], v[1]);
                        sq0 = fma(v[0], v[0], sq0);
                        sq1 = fma(v[1], v[1], sq1);
                    }
                    ua[i][0] = x[i][0];
                    ua[i][1] = x[i][1];
                }
            }
        }
        // per-shot |U|^2 of this warp's rows (lanes with equal lane & 3 hold the same shots); one
        // partial slot per team (k_ms_norms sums them in a fixed order)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            sq0 += __shfl_xor_sync(0xffffffffu, sq0, o);
            sq1 += __shfl_xor_sync(0xffffffffu, sq1, o);
        }
        if (lane < 4) {
            double* np = p.norm_part + (((size_t)kk * gridDim.x + blockIdx.x) * M4_NT + team) * S + q0;
            np[0] = sq0;
            np[1] = sq1;
        }
        // probes of this team's subdomains (this warp's 8 shots): rows of U after the step
        if (k % p.record_every == 0 && p.rows) {
            __syncwarp();
            const long long row = k / p.record_every - 1;
            const int q = 8 * cw + (lane & 7);
            for (int sl = team; sl < ns; sl += M4_NT) {
                const int s = s0 + sl;
                const double* us = Un + (size_t)s * KS;
                for (int pq = p.prb_ptr[s] + (lane >> 3); pq < p.prb_ptr[s + 1]; pq += 4) {
                    const int pid = p.prb_ids[pq];
                    const int tap = p.prb_tap[pid];
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
        // this step's state writes feed the next step's TMA reads (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(stepdone);
    }
#ifdef SFW_MS_CLK
    clk[3] = clock64() - clk_start;
    if (lane < 8 && p.dbg) {
        long long v = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (lane == i) v = clk[i];
        p.dbg[(blockIdx.x * M2_NW + 4 * team + cw) * 8 + lane] = v;
    }
#endif
#undef M4_T0
#undef M4_T1
}

template <int M>
__global__ void __launch_bounds__((M4_NW + 2 * M4_NT) * 32, 1) k_step_ms4(const MsParams p) {
    constexpr int S = 32;
    constexpr int RT = (6 * M + 7) / 8;
    constexpr int WP = 8 * RT;
    constexpr int W = 6 * M;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = p.L, TB = p.TB;
    const long long K = p.K;
    const long long WS = (long long)W * S, KS = K * S;
    double* cst = reinterpret_cast<double*>(smem_raw);          // [NT][NC][TB]
    double* sst = cst + (size_t)M4_NT * M4_NC * TB;             // [NT][NSS][W*S]
    double* Xall = sst + (size_t)M4_NT * M4_NSS * WS;           // [NW][WP][LDX]
    uint64_t* bars = reinterpret_cast<uint64_t*>(Xall + (size_t)M4_NW * WP * M4_LDX);
    // per team: cfull[NC], cempty[NC], sfull[NSS], sempty[NSS], stepdone
    constexpr int NB = 2 * M4_NC + 2 * M4_NSS + 1;
    int* ssub = reinterpret_cast<int*>(bars + M4_NT * NB);
    int* s_nb = ssub + S;  // [ns][6]

    for (int q = threadIdx.x; q < S; q += blockDim.x) ssub[q] = p.shot_sub[q];
    if (threadIdx.x == 0) {
        for (int t = 0; t < M4_NT; ++t) {
            uint64_t* b = bars + t * NB;
            for (int i = 0; i < M4_NC; ++i) {
                mbar_init(&b[i], 1);
                mbar_init(&b[M4_NC + i], 4);
            }
            for (int i = 0; i < M4_NSS; ++i) {
                mbar_init(&b[2 * M4_NC + i], 1);
                mbar_init(&b[2 * M4_NC + M4_NSS + i], 4);
            }
            mbar_init(&b[NB - 1], 4);
        }
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < M4_NW * WP * M4_LDX; i += blockDim.x) Xall[i] = 0.0;
    const int s0 = p.cta_sub_ptr[blockIdx.x], s1 = p.cta_sub_ptr[blockIdx.x + 1];
    const int ns = s1 - s0;
    for (int i = threadIdx.x; i < ns * 6; i += blockDim.x) s_nb[i] = p.nbr[s0 * 6 + i];
    __syncthreads();

    if (warp >= M4_NW) {  // producer warps: (team, ring) = ((warp - NW) / 2, (warp - NW) % 2)
        const int pw = warp - M4_NW, team = pw >> 1;
        uint64_t* b = bars + team * NB;
        uint64_t *cfull = b, *cempty = b + M4_NC, *sfull = b + 2 * M4_NC, *sempty = b + 2 * M4_NC + M4_NSS,
                 *stepdone = b + NB - 1;
        double* tc = cst + (size_t)team * M4_NC * TB;
        double* ts = sst + (size_t)team * M4_NSS * WS;
        if (lane != 0) return;
        if ((pw & 1) == 0) {  // chain-block ring of this team (ungated)
            const uint64_t pol = l2_policy_evict_first();
            const uint32_t cbytes = (uint32_t)TB * 8u;
            long long c_iss = 0;
            auto issue = [&](int sl, int bk) {
                const int st = (int)(c_iss % M4_NC);
                mbar_wait_sleep(&cempty[st], (uint32_t)(((c_iss / M4_NC) & 1) ^ 1));
                mbar_arrive_expect_tx(&cfull[st], cbytes);
                bulk_g2s(tc + (size_t)st * TB, p.tcoef + ((long long)(s0 + sl) * 2 * L + bk) * TB, cbytes, &cfull[st],
                         pol);
                ++c_iss;
            };
            for (int k = 0; k < p.n_steps; ++k) {
                for (int sl = team; sl < ns; sl += M4_NT) {  // A: G_0 [, H_0 on boundary subdomains]
                    const bool interior = s_nb[sl * 6] >= 0 && s_nb[sl * 6 + 1] >= 0 && s_nb[sl * 6 + 2] >= 0 &&
                                          s_nb[sl * 6 + 3] >= 0 && s_nb[sl * 6 + 4] >= 0 && s_nb[sl * 6 + 5] >= 0;
                    issue(sl, 0);
                    if (!interior) issue(sl, 1);
                }
                for (int sl = team; sl < ns; sl += M4_NT)  // B: G_j, H_j, j >= 1
                    for (int bk = 2; bk < 2 * L; ++bk) issue(sl, bk);
            }
        } else {  // state-block ring of this team, gated per step on the team's stepdone
            const uint64_t pol = l2_policy_evict_first();
            const uint32_t mbytes = (uint32_t)(6 * M * M * 8);
            const uint32_t sbytes = (uint32_t)(WS * 8);
            long long s_iss = 0;
            auto issue = [&](const double* src, uint32_t bytes) {
                const int st = (int)(s_iss % M4_NSS);
                mbar_wait_sleep(&sempty[st], (uint32_t)(((s_iss / M4_NSS) & 1) ^ 1));
                mbar_arrive_expect_tx(&sfull[st], bytes);
                bulk_g2s(ts + (size_t)st * WS, src, bytes, &sfull[st], pol);
                ++s_iss;
            };
            for (int k = 0; k < p.n_steps; ++k) {
                if (k > 0) mbar_wait_sleep(stepdone, (uint32_t)((k - 1) & 1));  // step k reads step k-1's output
                const int cbuf = k & 1;
                const double* cur = cbuf ? p.U1 : p.U0;
                const double* prv = cbuf ? p.U0 : p.U1;
                for (int sl = team; sl < ns; sl += M4_NT) {  // A: U_0, U_1
                    const long long base = (long long)(s0 + sl) * KS;
                    issue(cur + base, sbytes);
                    issue(cur + base + WS, sbytes);
                }
                for (int sl = team; sl < ns; sl += M4_NT) {  // C: U_0, Uprev_0, mass; B: U_1, [U_{j+1}], Uprev_j
                    const long long base = (long long)(s0 + sl) * KS;
                    issue(cur + base, sbytes);
                    issue(prv + base, sbytes);
                    issue(p.mblk + (size_t)(s0 + sl) * 6 * M * M, mbytes);
                    issue(cur + base + WS, sbytes);
                    for (int j = 1; j < L; ++j) {
                        if (j + 1 < L) issue(cur + base + (j + 1) * WS, sbytes);
                        issue(prv + base + j * WS, sbytes);
                    }
                }
            }
        }
        return;
    }
    const int team = warp / 4, cw = warp % 4;
    uint64_t* b = bars + team * NB;
    ms4_compute<M>(p, cst + (size_t)team * M4_NC * TB, sst + (size_t)team * M4_NSS * WS,
                   Xall + (size_t)warp * WP * M4_LDX, b, b + M4_NC, b + 2 * M4_NC, b + 2 * M4_NC + M4_NSS, b + NB - 1,
                   ssub, s_nb, s0, ns, team, cw, lane);
    (void)K;
}

static size_t ms4_smem_bytes(int RT, int TB, int W, int nsmax) {
    return 8 * ((size_t)M4_NT * M4_NC * TB + (size_t)M4_NT * M4_NSS * W * 32 + (size_t)M4_NW * 8 * RT * M4_LDX +
                (size_t)M4_NT * (2 * M4_NC + 2 * M4_NSS + 1)) +
           4 * (32 + 6 * (size_t)nsmax) + 64;
}

// ---------------------------------------------------------------------------
// k_step_ms3: shot-group-per-warp multi-shot stepping.  The 32 shots are 4
// independent groups of 8; warp (g, c) sweeps the layers of its subdomain group g
// (subdomains s0+g, s0+g+NG, ...) for shots 8c..8c+7 alone, so no warp ever waits
// for another inside a sweep.  Each block product is computed transposed,
//     (B X)^T = X^T B      (B symmetric: the stored lower tiles serve as the DMMA B operand),
// with the 8 x 4 X^T fragments built from the lane's own rows by two quad shuffles,
// and the result lands in the same row layout as the input (lane (q, a) holds rows
// 8I + 2a + {0,1} of shot q): the state, the fluxes and the accumulations of a sweep
// stay in registers.  The four warps of a group consume the same chain block from a
// shared TMA ring (full/empty mbarriers, 4 consumer arrivals per stage) fed by one
// producer warp; H_0 is streamed and applied only for subdomains with outer faces
// (the only rows of H_0 F_0 the step reads).  Layer-0 coupling waits on a per
// (subdomain, shot group) tagged flag of the neighbour's F_0 instead of a CTA flag.

__device__ __forceinline__ void mbar_wait_all(uint64_t* bar, uint32_t parity) {
    while (!__all_sync(0xffffffffu, mbar_try_wait(bar, parity))) {
    }
}

// C = (B X)^T for this lane's shot, X = P - Q (SUB) or P, given row-wise: lane (shot, a)
// holds rows 8I + 2a + {0,1}.  Two quad shuffles build each 8 x 4 X^T fragment.
template <int RT, bool SUB>
__device__ __forceinline__ void ms3_gemm(const double* __restrict__ tiles, const double (&P)[RT][2],
                                         const double (&Q)[RT][2], double (&C)[RT][2], int lane, int src_lo,
                                         int src_hi, const int (&tr)[2]) {
#pragma unroll
    for (int I = 0; I < RT; ++I) C[I][0] = C[I][1] = 0.0;
    const bool odd = (lane & 1) != 0;
#pragma unroll
    for (int kap = 0; kap < 2 * RT; ++kap) {
        const int Ip = kap >> 1, h = kap & 1;
        const double d0 = SUB ? P[Ip][0] - Q[Ip][0] : P[Ip][0];
        const double d1 = SUB ? P[Ip][1] - Q[Ip][1] : P[Ip][1];
        const int src = h ? src_hi : src_lo;
        const double v0 = __shfl_sync(0xffffffffu, d0, src);
        const double v1 = __shfl_sync(0xffffffffu, d1, src);
        const double xa = odd ? v1 : v0;
#pragma unroll
        for (int I = 0; I < RT; ++I) {
            const double b = (I >= Ip) ? tiles[(I * (I + 1) / 2 + Ip) * 64 + h * 32 + lane]
                                       : tiles[(Ip * (Ip + 1) / 2 + I) * 64 + tr[h]];
            dmma8x8x4(C[I], xa, b);
        }
    }
}

template <int M, int NG, int NSTG>
__global__ void __launch_bounds__(NG * 128, 1) k_step_ms3(const MsParams p) {
    constexpr int S = 32;
    constexpr int W = 6 * M;
    constexpr int RT = (W + 7) / 8;
    constexpr int NK = 2 * RT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = p.L, TB = p.TB;
    const long long K = p.K;
    const long long WS = (long long)W * S, KS = K * S;
    double* cst = reinterpret_cast<double*>(smem_raw);              // [NG][NS][TB]
    double* Tall = cst + (size_t)NG * NSTG * TB;                // [NCW][W][8] face sums (phase C)
    double* Sall = Tall + (size_t)(4 * NG) * W * 8;                  // [NCW][2][2 RT][32] staged state rows
    double* Mall = Sall + (size_t)(4 * NG) * 2 * 2 * RT * 32;         // [NCW][6 M M] interface mass of the next coupling
    uint64_t* full = reinterpret_cast<uint64_t*>(Mall + (size_t)(4 * NG) * 6 * M * M);
    uint64_t* empty = full + NG * NSTG;
    int* s_out = reinterpret_cast<int*>(empty + NG * NSTG);     // [ns] subdomain has an outer face
    const int s0 = p.cta_sub_ptr[blockIdx.x], s1 = p.cta_sub_ptr[blockIdx.x + 1];
    const int ns = s1 - s0;
    for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        int o = 0;
        for (int f = 0; f < 6; ++f) o |= p.nbr[(s0 + i) * 6 + f] < 0;
        s_out[i] = o;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < NG * NSTG; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 4);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // ======== compute warps ========
    const int g = warp >> 2, c = warp & 3;
    const int a = lane & 3;
    const int q = 8 * c + (lane >> 2);   // this lane's shot
    const int src_lo = (lane & ~3) | (a >> 1), src_hi = src_lo | 2;
    int tr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = 4 * h + a, cc = lane >> 2;
        tr[h] = (cc >> 2) * 32 + r * 4 + (cc & 3);
    }
    double* T = Tall + (size_t)warp * W * 8;
    // lane-private staging of the next layer's U_{j+2} and this layer's Uprev_j (cp.async, 8 B per row)
    double* sU = Sall + (size_t)warp * 2 * 2 * RT * 32;
    double* sP = sU + 2 * RT * 32;
#pragma unroll
    for (int i = 0; i < 2 * RT; ++i) sU[i * 32 + lane] = sP[i * 32 + lane] = 0.0;  // padding rows stay 0
    auto stage_rows = [&](const double* blk, double* dst) {
#pragma unroll
        for (int I = 0; I < RT; ++I)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = 8 * I + 2 * (lane & 3) + e;
                if (r < W)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst + (2 * I + e) * 32 + lane)),
                                 "l"(blk + (size_t)r * 32 + 8 * c + (lane >> 2))
                                 : "memory");
            }
    };
    // interface mass blocks of a subdomain -> this warp's SMEM copy (cp.async, 16 B per lane-op)
    double* Mw = Mall + (size_t)warp * 6 * M * M;
    auto stage_mass = [&](int sl) {
        const double* src = p.mblk + (size_t)(s0 + sl) * 6 * M * M;
        for (int i = lane; i < 3 * M * M; i += 32)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(Mw + 2 * i)), "l"(src + 2 * i)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto read_rows = [&](const double* src, double (&v)[RT][2]) {
#pragma unroll
        for (int I = 0; I < RT; ++I)
#pragma unroll
            for (int e = 0; e < 2; ++e) v[I][e] = src[(2 * I + e) * 32 + lane];
    };
    // chain-block ring of the group: warp c == 0 of the group refills it (lane 0 issues)
    // whenever all four consumers have released a stage -- at its own releases and while
    // it waits, so the ring never stalls on a refill nobody is in a position to make.
    long long con = 0, iss = 0, tot = 0;
    int pt = 0, pj = 0, ph = 0;
    if (c == 0) {
        long long per = 0;
        for (int sl = g; sl < ns; sl += NG) per += 2 * L - (s_out[sl] ? 0 : 1);
        tot = per * p.n_steps;
    }
    const uint64_t pol = l2_policy_evict_first();
    auto try_issue = [&]() {
        while (iss < tot) {
            const int st = (int)(iss % NSTG);
            uint64_t* e = &empty[g * NSTG + st];
            const int fr0 = lane == 0 ? (int)mbar_test_wait(e, (uint32_t)(((iss / NSTG) & 1) ^ 1)) : 0;
            if (!__shfl_sync(0xffffffffu, fr0, 0)) break;
            const int sl = g + pt * NG;
            if (lane == 0) {
                const long long blk = (long long)(s0 + sl) * 2 * L + 2 * pj + ph;
                uint64_t* fb = &full[g * NSTG + st];
                mbar_arrive_expect_tx(fb, (uint32_t)TB * 8u);
                bulk_g2s(cst + (size_t)(g * NSTG + st) * TB, p.tcoef + blk * TB, (uint32_t)TB * 8u, fb, pol);
            }
            ++iss;
            if (ph == 0 && (pj > 0 || s_out[sl])) {  // G_j, H_j per layer; H_0 only with an outer face
                ph = 1;
            } else {
                ph = 0;
                if (++pj == L) {
                    pj = 0;
                    if (g + (++pt) * NG >= ns) pt = 0;
                }
            }
        }
    };
    if (c == 0) try_issue();
    // optional cycle accounting (p.dbg, SFW_STEP_PROF): [acquire wait, gemm, coupling, total]
    const bool prof = p.dbg != nullptr;
    long long clk_acq = 0, clk_gemm = 0, clk_coup = 0, clk_wait = 0, clk_f0 = 0;
    const long long clk_start = prof ? clock64() : 0;
    auto acquire = [&]() -> const double* {
        const int st = (int)(con % NSTG);
        uint64_t* fb = &full[g * NSTG + st];
        const uint32_t par = (uint32_t)((con / NSTG) & 1);
        const long long t0 = prof ? clock64() : 0;
        while (!__all_sync(0xffffffffu, mbar_try_wait(fb, par)))
            if (c == 0) try_issue();
        if (prof) clk_acq += clock64() - t0;
        return cst + (size_t)(g * NSTG + st) * TB;
    };
    auto release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[g * NSTG + (con % NSTG)]);
        ++con;
        if (c == 0) try_issue();
    };
    auto row_of = [&](int I, int e) { return 8 * I + 2 * a + e; };
    auto load_rows = [&](const double* blk, double (&v)[RT][2]) {  // blk: [W][S] layer block
#pragma unroll
        for (int I = 0; I < RT; ++I)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = row_of(I, e);
                v[I][e] = r < W ? blk[(size_t)r * S + q] : 0.0;
            }
    };
    const double dt2 = p.dt2;
    const int ssq = p.shot_sub[q];
    const double* svec = p.shot_vec + p.shot_voff[q];
    const int n_g = ns > g ? (ns - g + NG - 1) / NG : 0;
    const int NWG = gridDim.x * NG;
    auto buf = [&](int lvl) -> double* { return (lvl & 1) ? p.U1 : p.U0; };  // level n lives in buf(n)
    auto ftab_of = [&](int kk) -> double { return ssq >= 0 ? p.ftab[(size_t)q * p.ftab_stride + kk] : 0.0; };

    // Layer-0 coupling of step kc (level kc): shared faces mass (own + neighbour F_0), outer
    // faces acc_0, leapfrog.  Result rows also returned in u0n (the next sweep's U_0).
    auto coupling = [&](int kc, int t, double (&u0n)[RT][2], double& sqc) {
        const int sl = g + t * NG, s = s0 + sl;
        const unsigned int tag = p.tag0 + (unsigned int)kc;
        const double* fx = p.flux + (size_t)(tag & 1u) * p.n_sub * WS;
        const double* uc = buf(kc - 1) + (size_t)s * KS;   // level kc-1
        double* un = buf(kc) + (size_t)s * KS;             // level kc-2 on entry (layer 0), kc on exit
        const bool srcs = ssq == s;
        const double fq = ftab_of(kc - 1);
        double u0[RT][2];
        load_rows(uc, u0);
        load_rows(un, u0n);  // Uprev_0 (overwritten below)
        {   // neighbours' F_0 of this shot group: tags are monotone, a neighbour may be a step ahead
            const int nb = lane < 6 ? p.nbr[s * 6 + lane] : -1;
            int spins = 0;
            while (!__all_sync(0xffffffffu, nb < 0 || (int)(ld_acquire(p.sflags + (size_t)nb * 4 + c) - tag) >= 0))
                if (++spins > 2) __nanosleep(64);
            __syncwarp();  // the acquiring lanes' view of the neighbours' F_0 -> every lane
        }
        const double* fo = fx + (size_t)s * WS;
#pragma unroll
        for (int I = 0; I < RT; ++I)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = row_of(I, e);
                if (r < W) {
                    const int f = r / M, cm = r % M, nb = p.nbr[s * 6 + f];
                    if (nb >= 0) {
                        const double own = __ldcg(fo + (size_t)r * S + q);
                        const double oth = __ldcg(fx + ((size_t)nb * W + (f ^ 1) * M + cm) * S + q);
                        T[r * 8 + (lane >> 2)] = __dadd_rn(own, oth);
                    }
                }
            }
        __syncwarp();
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();  // Mw (staged by every lane) visible to the warp
#pragma unroll
        for (int I = 0; I < RT; ++I)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = row_of(I, e);
                double v = 0.0;
                if (r < W) {
                    const int f = r / M, rr = r % M;
                    double acc;
                    if (p.nbr[s * 6 + f] >= 0) {
                        acc = 0.0;
                        const double* mx = Mw + (f * M + rr) * M;
                        const double* tx = T + (f * M) * 8 + (lane >> 2);
#pragma unroll
                        for (int cm = 0; cm < M; ++cm) acc = fma(mx[cm], tx[cm * 8], acc);
                    } else {
                        acc = __ldcg(p.acc1 + ((size_t)s * W + r) * S + q);
                    }
                    if (srcs) acc = __dadd_rn(acc, __dmul_rn(svec[r], fq));
                    v = __dadd_rn(__dsub_rn(__dmul_rn(2.0, u0[I][e]), u0n[I][e]), __dmul_rn(dt2, acc));
                    un[(size_t)r * S + q] = v;
                    sqc = fma(v, v, sqc);
                }
                u0n[I][e] = v;
            }
        __syncwarp();
    };
    // probe rows of level kc for subdomain slot t (all its layers are final)
    auto probes = [&](int kc, int t) {
        if (kc % p.record_every != 0 || !p.rows) return;
        const int s = s0 + g + t * NG;
        if (p.prb_ptr[s] == p.prb_ptr[s + 1]) return;
        const long long row = kc / p.record_every - 1;
        const int qp = 8 * c + (lane & 7), part = lane >> 3;
        const double* us = buf(kc) + (size_t)s * KS;
        for (int pq = p.prb_ptr[s]; pq < p.prb_ptr[s + 1]; ++pq) {
            const int pid = p.prb_ids[pq];
            const int tap = p.prb_tap[pid];
            double val = 0.0;
            if (tap >= 0) {
                val = part == 0 ? us[(size_t)tap * S + qp] : 0.0;
            } else {
                const double* wv = p.prb_w + p.prb_woff[pid];
                for (long long i0 = 0; i0 < K; i0 += 4) {
                    const long long i = i0 + part;
                    if (i < K) val = fma(wv[i], us[i * S + qp], val);
                }
            }
            val += __shfl_xor_sync(0xffffffffu, val, 8);
            val += __shfl_xor_sync(0xffffffffu, val, 16);
            if (part == 0) p.rows[(row * p.n_probe + pid) * S + qp] = val;
        }
        __syncwarp();
    };
    auto put_norm = [&](int kc, double v) {  // per-shot |U|^2 of level kc (the quad's 4 lanes share a shot)
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (a == 0) p.norm_part[((size_t)(kc - 1) * NWG + blockIdx.x * NG + g) * S + q] = v;
    };

    // Iteration k: for every subdomain of the group, the layer-0 coupling of step k-1 (its
    // neighbours published F_0 during the previous sweep, so the flags are normally set)
    // immediately followed by the sweep of step k, which takes the new U_0 from registers.
    double sq_prev = 0.0;  // |U|^2 of the previous step's layers >= 1
    if (n_g > 0) stage_mass(g);
    for (int k = 1; k <= p.n_steps + 1; ++k) {
        const bool sweep = k <= p.n_steps;
        const unsigned int tag = p.tag0 + (unsigned int)k;
        double* fx = p.flux + (size_t)(tag & 1u) * p.n_sub * WS;
        const double* Uc = buf(k - 1);   // level k-1
        double* Un = buf(k);             // level k-2 -> k
        const double fq = ftab_of(k - 1);
        double sq = 0.0, sqc = 0.0;
        for (int t = 0; t < n_g; ++t) {
            const int sl = g + t * NG, s = s0 + sl;
            const bool outer = s_out[sl] != 0;
            const bool srcs = ssq == s;
            const double* us = Uc + (size_t)s * KS;
            double* un = Un + (size_t)s * KS;
            double Uj[RT][2], Uj1[RT][2], Fp[RT][2], C[RT][2];
            if (sweep) load_rows(us + WS, Uj1);  // U_1 of level k-1 (in flight during the coupling)
            if (k > 1) {
                const long long tc_ = prof ? clock64() : 0;
                coupling(k - 1, t, Uj, sqc);
                probes(k - 1, t);
                if (prof) clk_coup += clock64() - tc_;
                stage_mass(g + ((t + 1) % n_g) * NG);  // next coupling's mass, in flight during the sweep
            } else {
                load_rows(us, Uj);
            }
            if (!sweep) continue;
            for (int j = 0; j < L; ++j) {
                // stage U_{j+2} (level k-1) and Uprev_j (level k-2) while the two products run
                if (j + 2 < L) stage_rows(us + (size_t)(j + 2) * WS, sU);
                if (j > 0) stage_rows(un + (size_t)j * WS, sP);
                asm volatile("cp.async.commit_group;" ::: "memory");
                // F_j = G_j (U_{j+1} - U_j)
                {
                    const double* tl_ = acquire();
                    const long long tg_ = prof ? clock64() : 0;
                    ms3_gemm<RT, true>(tl_, Uj1, Uj, C, lane, src_lo, src_hi, tr);
                    if (prof) clk_gemm += clock64() - tg_;
                }
                release();
                if (j == 0) {
                    // F_0 -> face mailbox (all W rows are face rows), then the per-warp flag
                    const long long tf_ = prof ? clock64() : 0;
                    double* fo = fx + (size_t)s * WS;
#pragma unroll
                    for (int I = 0; I < RT; ++I)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int r = row_of(I, e);
                            if (r < W) fo[(size_t)r * S + q] = C[I][e];
                        }
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) st_release(p.sflags + (size_t)s * 4 + c, tag);
                    if (prof) clk_f0 += clock64() - tf_;
                    if (outer) {  // acc_0 = H_0 F_0 (read back only on outer-face rows)
                        double A0[RT][2];
                        {
                            const double* tl_ = acquire();
                            const long long tg_ = prof ? clock64() : 0;
                            ms3_gemm<RT, false>(tl_, C, C, A0, lane, src_lo, src_hi, tr);
                            if (prof) clk_gemm += clock64() - tg_;
                        }
                        release();
                        double* ao = p.acc1 + (size_t)s * WS;
#pragma unroll
                        for (int I = 0; I < RT; ++I)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int r = row_of(I, e);
                                if (r < W && p.nbr[s * 6 + r / M] < 0) ao[(size_t)r * S + q] = A0[I][e];
                            }
                    }
#pragma unroll
                    for (int I = 0; I < RT; ++I) {
                        Fp[I][0] = C[I][0];
                        Fp[I][1] = C[I][1];
                    }
                } else {
                    // acc_j = H_j (F_j - F_{j-1}); leapfrog of layer j
                    double A[RT][2];
                    {
                        const double* tl_ = acquire();
                        const long long tg_ = prof ? clock64() : 0;
                        ms3_gemm<RT, true>(tl_, C, Fp, A, lane, src_lo, src_hi, tr);
                        if (prof) clk_gemm += clock64() - tg_;
                    }
                    release();
                    {
                        const long long tw_ = prof ? clock64() : 0;
                        asm volatile("cp.async.wait_group 0;" ::: "memory");
                        if (prof) clk_wait += clock64() - tw_;
                    }
#pragma unroll
                    for (int I = 0; I < RT; ++I)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int r = row_of(I, e);
                            double tot = A[I][e];
                            if (srcs && r < W) tot = __dadd_rn(tot, __dmul_rn(svec[(size_t)j * W + r], fq));
                            const double upr = sP[(2 * I + e) * 32 + lane];
                            const double v =
                                __dadd_rn(__dsub_rn(__dmul_rn(2.0, Uj[I][e]), upr), __dmul_rn(dt2, tot));
                            if (r < W) {
                                un[(size_t)j * WS + (size_t)r * S + q] = v;
                                sq = fma(v, v, sq);
                            }
                            Fp[I][e] = C[I][e];
                        }
                }
                {
                    const long long tw_ = prof ? clock64() : 0;
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                    if (prof) clk_wait += clock64() - tw_;
                }
#pragma unroll
                for (int I = 0; I < RT; ++I)
#pragma unroll
                    for (int e = 0; e < 2; ++e) Uj[I][e] = Uj1[I][e];
                if (j + 2 < L) {
                    read_rows(sU, Uj1);
                } else {
#pragma unroll
                    for (int I = 0; I < RT; ++I) Uj1[I][0] = Uj1[I][1] = 0.0;
                }
            }
        }
        if (k > 1) put_norm(k - 1, sq_prev + sqc);
        sq_prev = sq;
        __syncwarp();
    }
    if (prof && lane < 6) {
        const long long v = lane == 0 ? clk_acq : lane == 1 ? clk_gemm : lane == 2 ? clk_coup
                          : lane == 3 ? clock64() - clk_start : lane == 4 ? clk_wait : clk_f0;
        p.dbg[(blockIdx.x * (4 * NG) + warp) * 8 + lane] = (unsigned long long)v;
    }
}

static size_t ms3_smem_bytes(int TB, int W, int nsmax, int ng, int nstg) {
    const size_t RT = (W + 7) / 8, M = W / 6;
    return 8 * ((size_t)ng * nstg * TB + (size_t)4 * ng * W * 8 + (size_t)4 * ng * 4 * RT * 32 +
                (size_t)4 * ng * 6 * M * M + 2 * ng * nstg) +
           4 * (size_t)nsmax + 64;
}

// launch shapes of k_step_ms3: (subdomain groups per CTA, chain stages per group)
static const void* ms3_kernel(int m, int ng, int nstg) {
#define SFW_MS3_CASE(MM, G, NSV) \
    if (m == MM && ng == G && nstg == NSV) return (const void*)k_step_ms3<MM, G, NSV>;
    SFW_MS3_CASE(9, 2, 3)
    SFW_MS3_CASE(4, 2, 3)
    SFW_MS3_CASE(1, 2, 3)
#undef SFW_MS3_CASE
    return nullptr;
}

// per-subdomain interface mass blocks [n_sub][6][m*m] (zeros on outer faces)
__global__ void k_ms_massblocks(const double* __restrict__ mass, const int* __restrict__ mass_idx, int n_sub, int m,
                                double* __restrict__ out) {
    const long long total = (long long)n_sub * 6 * m * m;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long sf = i / (m * m);
        const int e = (int)(i % (m * m));
        const int mi = mass_idx[sf];
        out[i] = mi >= 0 ? mass[(size_t)mi * m * m + e] : 0.0;
    }
}

static const void* ms2_kernel(int m) {
    static const void* const tab[10] = {nullptr,
                                        (const void*)k_step_ms2<1>,
                                        (const void*)k_step_ms2<2>,
                                        (const void*)k_step_ms2<3>,
                                        (const void*)k_step_ms2<4>,
                                        (const void*)k_step_ms2<5>,
                                        (const void*)k_step_ms2<6>,
                                        (const void*)k_step_ms2<7>,
                                        (const void*)k_step_ms2<8>,
                                        (const void*)k_step_ms2<9>};
    return (m >= 1 && m <= 9) ? tab[m] : nullptr;
}

static const void* ms4_kernel(int m) {
    static const void* const tab[10] = {nullptr,
                                        (const void*)k_step_ms4<1>,
                                        (const void*)k_step_ms4<2>,
                                        (const void*)k_step_ms4<3>,
                                        (const void*)k_step_ms4<4>,
                                        (const void*)k_step_ms4<5>,
                                        (const void*)k_step_ms4<6>,
                                        (const void*)k_step_ms4<7>,
                                        (const void*)k_step_ms4<8>,
                                        (const void*)k_step_ms4<9>};
    return (m >= 1 && m <= 9) ? tab[m] : nullptr;
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
    if (ms2_kernel(h->m) && !getenv("SFW_MS_V1")) {
        const void* k2 = ms2_kernel(h->m);
        int nsmax = 0;
        for (int b = 0; b < h->grid; ++b) nsmax = std::max(nsmax, h->cta_ptr_h[b + 1] - h->cta_ptr_h[b]);
        h->shot_smem2 = (int)ms2_smem_bytes(RT, h->TB, W, nsmax);
        if (!h->mmass && (rc = dalloc(&h->mmass, (size_t)h->n_sub * 6 * h->m * h->m, errbuf, errlen))) return rc;
        k_ms_massblocks<<<592, 256, 0, h->stream>>>(h->mass, h->mass_idx, h->n_sub, h->m, h->mmass);
        if (h->shot_smem2 <= 220 * 1024)
            SFW_CUDA_TRY(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, h->shot_smem2));
        else
            h->shot_smem2 = 0;
    } else {
        h->shot_smem2 = 0;
    }
    h->shot_smem4 = 0;
    if (ms4_kernel(h->m) && getenv("SFW_MS4")) {  // opt-in two-team kernel (measured slower)
        int nsmax = 0;
        for (int b = 0; b < h->grid; ++b) nsmax = std::max(nsmax, h->cta_ptr_h[b + 1] - h->cta_ptr_h[b]);
        const size_t sm4 = ms4_smem_bytes(RT, h->TB, W, nsmax);
        if (!h->mmass && (rc = dalloc(&h->mmass, (size_t)h->n_sub * 6 * h->m * h->m, errbuf, errlen))) return rc;
        k_ms_massblocks<<<592, 256, 0, h->stream>>>(h->mass, h->mass_idx, h->n_sub, h->m, h->mmass);
        if (sm4 <= 227 * 1024) {
            SFW_CUDA_TRY(cudaFuncSetAttribute(ms4_kernel(h->m), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4));
            h->shot_smem4 = (int)sm4;
        }
    }
    h->shot_smem3 = 0;
    // k_step_ms3 is opt-in (SFW_MS3="groups,stages", e.g. "2,3"): correct, but measured slower than
    // k_step_ms2 on config 4 (0.93 vs 0.79 ms/step): with 2 warps per SMSP the in-sweep layer-0
    // coupling (three dependent global round trips per subdomain) leaves the DMMA pipe idle.
    int ng = 0, nstg = 0;
    if (const char* e = getenv("SFW_MS3")) sscanf(e, "%d,%d", &ng, &nstg);
    if (ng > 0 && ms3_kernel(h->m, ng, nstg) && !getenv("SFW_MS_V1")) {
        int nsmax = 0;
        for (int b = 0; b < h->grid; ++b) nsmax = std::max(nsmax, h->cta_ptr_h[b + 1] - h->cta_ptr_h[b]);
        const size_t sm3 = ms3_smem_bytes(h->TB, W, nsmax, ng, nstg);
        h->ms3_ng = ng;
        h->ms3_ns = nstg;
        if (!h->mmass && (rc = dalloc(&h->mmass, (size_t)h->n_sub * 6 * h->m * h->m, errbuf, errlen))) return rc;
        k_ms_massblocks<<<592, 256, 0, h->stream>>>(h->mass, h->mass_idx, h->n_sub, h->m, h->mmass);
        if (!h->sflags) {
            if ((rc = dalloc(&h->sflags, (size_t)h->n_sub * 4, errbuf, errlen))) return rc;
            SFW_CUDA_TRY(cudaMemsetAsync(h->sflags, 0, (size_t)h->n_sub * 4 * 4, h->stream));
            h->stag = 0;
        }
        if (sm3 <= 220 * 1024) {
            SFW_CUDA_TRY(cudaFuncSetAttribute(ms3_kernel(h->m, ng, nstg), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)sm3));
            h->shot_smem3 = (int)sm3;
        }
    }
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
    // norm partials per step: ms3 one per subdomain group, ms2 one per row-tile group, ms one per CTA
    const int nparts = h->shot_smem4   ? M4_NT * h->grid
                       : h->shot_smem3 ? h->ms3_ng * h->grid
                       : h->shot_smem2 ? M2_NQ * h->grid
                                       : h->grid;
    if ((rc = ms_ensure(&h->mnorm, &h->mnorm_cap, (long long)n_steps * nparts * S + (long long)n_steps * S, errbuf,
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
    p.dbg = nullptr;
    p.mblk = h->mmass;
    if (getenv("SFW_STEP_PROF")) {
        const size_t need = (size_t)h->grid * M2_NW * 8;
        if (h->tprof_n < need) {
            if (h->tprof) cudaFree(h->tprof);
            cudaMalloc(&h->tprof, need * 8);
            h->tprof_n = need;
        }
        cudaMemsetAsync(h->tprof, 0, need * 8, h->stream);
        p.dbg = h->tprof;
    }
    void* args[] = {&p};
    SFW_CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
    p.sflags = h->sflags;
    p.tag0 = h->stag;
    if (h->shot_smem4) {
        SFW_CUDA_TRY(cudaLaunchCooperativeKernel(ms4_kernel(h->m), dim3(h->grid), dim3((M4_NW + 2 * M4_NT) * 32), args,
                                                 h->shot_smem4, h->stream));
    } else if (h->shot_smem3) {
        SFW_CUDA_TRY(cudaLaunchCooperativeKernel(ms3_kernel(h->m, h->ms3_ng, h->ms3_ns), dim3(h->grid),
                                                 dim3(128 * h->ms3_ng), args,
                                                 h->shot_smem3, h->stream));
        h->stag += (unsigned int)n_steps;
    } else if (h->shot_smem2)
        SFW_CUDA_TRY(cudaLaunchCooperativeKernel(ms2_kernel(h->m), dim3(h->grid), dim3((M2_NW + 2) * 32), args,
                                                 h->shot_smem2, h->stream));
    else
        SFW_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_step_ms<32>, dim3(h->grid), dim3((MS_NW + 1) * 32),
                                                 args, h->shot_smem, h->stream));
    SFW_CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
    double* dn = h->mnorm + (size_t)n_steps * nparts * S;
    k_ms_norms<<<(unsigned)((n_steps * S + 255) / 256), 256, 0, h->stream>>>(h->mnorm, n_steps, nparts, S, dn);
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
