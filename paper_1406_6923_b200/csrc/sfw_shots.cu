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
    double* rows;          // [n_rec][S][n_probe]
    double* norm_part;     // [n_steps][grid][S]
    unsigned int* flags;
    const int* ncta_ptr;
    const int* ncta;
    int evict_first;
    unsigned long long* dbg;  // debug cycle counters (SFW_MS_CLK builds) or null
    const double* mblk;       // [n_sub][6][M*M] interface mass per face (0 for outer faces)
};

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
constexpr int M2_NC = 4;    // chain-block stages (5 with a swizzled 8-wide X tile measured 4% slower)
constexpr int M2_NSS = 8;   // state-block stages
constexpr int M2_LDX = 12;  // padded X row stride (conflict-free fragment reads)
__device__ __forceinline__ int m2_xs(int row, int col) { return row * M2_LDX + col; }
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

    for (int k = 1; k <= p.n_steps; ++k) {
        const int par = k & 1;
        const int cb = (k - 1) & 1;
        double* Un = cb ? p.U0 : p.U1;
        double* fx = p.flux + (size_t)par * p.n_sub * WS;
        const int kk = k - 1;
        const double f0 = src0 ? p.ftab[(size_t)q0 * p.ftab_stride + kk] : 0.0;
        const double f1 = src1 ? p.ftab[(size_t)(q0 + 1) * p.ftab_stride + kk] : 0.0;
        double sq0 = 0.0, sq1 = 0.0;
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
                    p.rows[(row * S + q) * p.n_probe + pid] = val;  // [rec][shot][probe]
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
                        mbar_wait(&cempty[st], (uint32_t)(((c_iss / M2_NC) & 1) ^ 1));
                        mbar_arrive_expect_tx(&cfull[st], cbytes);
                        bulk_g2s(cst + (size_t)st * TB, p.tcoef + ((long long)(s0 + sl) * 2 * L + b) * TB, cbytes,
                                 &cfull[st], pol);
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
                if (k > 0) mbar_wait(stepdone, (uint32_t)((k - 1) & 1));
                const int cb = k & 1;
                const double* cur = cb ? p.U1 : p.U0;
                const double* prv = cb ? p.U0 : p.U1;
                for (int spos = 0; spos < ns * (nab + 3); ++spos) {
                    const double* src;
                    uint32_t bytes = sbytes;
                    if (spos < ns * nab) {
                        const int sl = spos / nab, r = spos % nab;
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
                        const int r = spos - ns * nab, sl = r / 3, w3 = r % 3;
                        if (w3 == 0) {  // interface mass of the 6 faces
                            src = p.mblk + (size_t)(s0 + sl) * 6 * M * M;
                            bytes = mbytes;
                        } else {
                            src = ((w3 == 2) ? prv : cur) + (long long)(s0 + sl) * KS;  // U_0, Uprev_0
                        }
                    }
                    const int st = (int)(s_iss % M2_NSS);
                    mbar_wait(&sempty[st], (uint32_t)(((s_iss / M2_NSS) & 1) ^ 1));
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
    if (L < 2) return fail(SFW_ECONFIG, "multi-shot stepping needs at least 2 layers", errbuf, errlen);
    if (!ms2_kernel(h->m))
        return fail(SFW_ECONFIG, "multi-shot stepping supports 1 <= modes per face <= 9", errbuf, errlen);
    {
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
    }
    if (!h->shot_smem2)
        return fail(SFW_ECONFIG, "multi-shot stepping: too many subdomains per CTA for the shared-memory rings",
                    errbuf, errlen);
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
    // norm partials per step: one per (CTA, row-tile group)
    const int nparts = M2_NQ * h->grid;
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
    SFW_CUDA_TRY(cudaLaunchCooperativeKernel(ms2_kernel(h->m), dim3(h->grid), dim3((M2_NW + 2) * 32), args,
                                             h->shot_smem2, h->stream));
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
