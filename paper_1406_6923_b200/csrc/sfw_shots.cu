// Multi-shot stepping (BASELINE config 4): S = 32 independent wavefields advanced in
// one persistent launch.  The reference runs one CoupledStepper per shot
// (stepper.py:144-449 with a single SourceTerm); here every chain
// block product Gamma_j X / Gamma-hat_j X over the shots is an fp64 GEMM on the DMMA pipe
// (mma.sync.m8n8k4.f64).
//
// Orientation.  The product is computed transposed, Y^T = X^T B (B symmetric): the shots
// are the M dimension of the MMA, the rows of the block its K and N dimensions.  The
// accumulator fragment of m8n8k4 gives lane l the elements (shot l/4, rows 8t + 2(l%4) + e),
// e = 0, 1, of row tile t; the A fragment of a k-step wants (shot l/4, k = l%4).  Numbering
// the k-steps kappa = 2T + e and letting position c of k-step kappa stand for row
// 8T + 2c + e makes the accumulator of one GEMM, element for element in the same lane, the
// A operand of the next: differences, leapfrog and the whole layer sweep of a subdomain
// stay with the warp.  One warp owns 8 shots of a subdomain and sweeps its layers alone; no
// X tile is exchanged through shared memory and no warp waits for another inside a sweep
// (the slices needed again after a product -- U_j, U_{j+1}, F_{j-1} -- rest in a warp-private
// shared-memory scratch while the GEMMs run).  The row permutation of the k-steps is folded
// into the stored chain blocks (the B operand).
//
// Chain block storage: the lower 8 x 8 tiles (T >= t) of the padded symmetric block, each
// tile's 64 doubles at the swizzled positions mt_pos(r, c), so that the B fragment of tile
// (T, t) -- element (2(l%4) + e, l/4) -- and that of its transpose -- element (l/4, 2(l%4) + e)
// of tile (t, T) -- are both conflict-free 8-byte shared loads.  A block is streamed once.
//
// Team = 4 compute warps (shots 8w .. 8w+7) + 1 producer warp; two teams per CTA, one CTA per
// SM.  One lane of the producer warp streams chain blocks and 32-shot state blocks, in the order the sweep
// consumes them, through a single ring of equal stages (cp.async.bulk + mbarrier).  Per step k:
//   sweep   per subdomain: first the DEFERRED layer 0 of step k-1 (k >= 2): T = F_0 + neighbour's F_0 of
//           step k-1 on shared faces, acc_0 = mass T as a GEMM over the tiles that meet a face block
//           (block-diagonal mass), leapfrog into the layer-0 slot of U^{k-1}; the new U_0 stays in
//           registers.  Then F_0 = G_0 (U_1 - U_0) -> face buffer (global); boundary subdomains also
//           acc_0 = H_0 F_0; layers j = 1..L-1: F_j, A_j = H_j (F_j - F_{j-1}), leapfrog
//   barrier team barrier, step flag (release), norms and the probes of step k-1, wait for the step flags
//           of ALL teams (acquire)
//   after the last step: one layer-0 pass for that step (epilogue).
// Folding the layer-0 pass into the next sweep (as k_ustep does) overlaps its 209 MB of traffic per
// step with the other warps' GEMMs and saves one U_0 read per subdomain-step; the face buffer is
// double-buffered by step parity and a team starts step k+1 only after every team finished sweep k, so a
// flux of step k-1 is never overwritten (by a sweep of step k+1) while a sweep of step k still reads it.
// State layout in HBM: [subdomain][layer][shot][WP rows] (rows padded to 8 RT, pad = 0), so a
// lane's two adjacent rows are one 16-byte access and a warp's 8 shots of a row tile are
// eight 64-byte segments.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>
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

// position of element (r, c) inside a stored 8 x 8 tile.  Over the 16 lanes of a half-warp the
// direct fragment {(2a + e, b)} and the transposed one {(b, 2a + e)}, a, b in 0..3, both hit 16
// distinct 8-byte banks (low four bits: r1, c1, r2 ^ c2, r0 ^ c0).
__host__ __device__ constexpr int mt_pos(int r, int c) {
    return 16 * (2 * (r >> 2) + (r & 1)) + 8 * ((r >> 1) & 1) + 4 * ((c >> 1) & 1) + 2 * ((r >> 2) ^ (c >> 2)) +
           ((r & 1) ^ (c & 1));
}

// does tile (T, t) of the block-diagonal interface mass (6 face blocks of m x m) hold a nonzero?
__host__ __device__ constexpr bool mt_face_tile(int m, int T, int t) {
    for (int f = 0; f < 6; ++f) {
        const int lo = f * m, hi = lo + m;
        if (lo < 8 * T + 8 && hi > 8 * T && lo < 8 * t + 8 && hi > 8 * t) return true;
    }
    return false;
}

// compact index of lower tile (T, t), T >= t, among the mass tiles (row-major lower order)
__host__ __device__ constexpr int mt_mass_idx(int m, int T, int t) {
    int n = 0;
    for (int I = 0; I <= T; ++I)
        for (int K = 0; K <= I; ++K) {
            if (I == T && K == t) return n;
            if (mt_face_tile(m, I, K)) ++n;
        }
    return n;
}

__host__ __device__ constexpr int mt_mass_count(int m) {
    const int RT = (6 * m + 7) / 8;
    int n = 0;
    for (int I = 0; I < RT; ++I)
        for (int K = 0; K <= I; ++K)
            if (mt_face_tile(m, I, K)) ++n;
    return n;
}

// 6-group packed blocks -> swizzled lower 8 x 8 tiles
__global__ void k_tilepack(const double* __restrict__ packed, int BS, int m, int RT, int TB,
                           double* __restrict__ out, long long n_blocks) {
    const long long b = blockIdx.x;
    if (b >= n_blocks) return;
    const int w = 6 * m;
    const double* src = packed + b * BS;
    double* dst = out + b * TB;
    const int ntl = RT * (RT + 1) / 2;
    for (int idx = threadIdx.x; idx < ntl * 64; idx += blockDim.x) {
        const int tl = idx / 64, within = idx % 64;
        int I = 0;
        while ((I + 1) * (I + 2) / 2 <= tl) ++I;
        const int K = tl - I * (I + 1) / 2;
        const int r = within / 8, c = within % 8;
        const int row = I * 8 + r, col = K * 8 + c;
        dst[tl * 64 + mt_pos(r, c)] = (row < w && col < w) ? src[ms_packed_pos(m, row, col)] : 0.0;
    }
}

// per-subdomain interface mass as swizzled tiles [n_sub][NMT][64] (zeros on outer faces; the mass
// of an interface is symmetric, stepper.py:209)
__global__ void k_mt_masstiles(const double* __restrict__ mass, const int* __restrict__ mass_idx, int n_sub, int m,
                               int RT, int NMT, double* __restrict__ out) {
    const int s = blockIdx.x;
    if (s >= n_sub) return;
    const int w = 6 * m;
    for (int I = 0; I < RT; ++I)
        for (int K = 0; K <= I; ++K) {
            if (!mt_face_tile(m, I, K)) continue;
            const int tl = mt_mass_idx(m, I, K);
            for (int e = threadIdx.x; e < 64; e += blockDim.x) {
                const int r = e / 8, c = e % 8, row = I * 8 + r, col = K * 8 + c;
                double v = 0.0;
                if (row < w && col < w && row / m == col / m) {
                    const int mi = mass_idx[s * 6 + row / m];
                    if (mi >= 0) v = mass[(size_t)mi * m * m + (row % m) * m + (col % m)];
                }
                out[((size_t)s * NMT + tl) * 64 + mt_pos(r, c)] = v;
            }
        }
}

struct MtParams {
    int n_sub, L, n_steps, record_every, n_probe, ftab_stride, nst;
    int n_team, team_smem;  // teams in the launch (two per CTA); shared-memory bytes of one team
    double dt2;
    const double* tcoef;   // [n_blocks][TB] swizzled lower tiles; block 2j = Gamma_j, 2j+1 = Gamma-hat_j
    const double* mtiles;  // [n_sub][NMT][64]
    double* U0;
    double* U1;            // [n_sub][L][S][WP]
    double* flux;          // [2][n_sub][S][WP] layer-0 flux F_0 (face mailbox), double-buffered by parity
    double* acc1;          // [n_sub][S][WP] H_0 F_0 of boundary subdomains
    const int* nbr;
    const int* cta_sub_ptr;  // [n_team + 1] offsets into team_subs
    const int* team_subs;    // subdomains of every team (ascending within a team)
    int nsmax;               // most subdomains in a team
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
    double* norm_part;     // [n_steps][2][n_team][S]  (slot 0: layers >= 1, slot 1: layer 0)
    unsigned int* flags;   // [n_team] step of the last finished sweep
};

constexpr int MT_NCW = 4;  // compute warps per CTA (8 shots each)

template <int M>
struct MtDims {
    static constexpr int S = 32;
    static constexpr int W = 6 * M;
    static constexpr int RT = (W + 7) / 8;
    static constexpr int WP = 8 * RT;
    static constexpr int TB = RT * (RT + 1) / 2 * 64;  // doubles per chain block
    static constexpr int SB = S * WP;                  // doubles per 32-shot state block
    static constexpr int STG = TB > SB ? TB : SB;      // ring stage (doubles)
    static constexpr int NMT = mt_mass_count(M);
};

// compile-time loop: f(std::integral_constant<int, 0>{}), ..., f(std::integral_constant<int, N - 1>{})
template <typename F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// B fragments of k-step KC (all row tiles): element for element what mt_gemm's MMAs of that k-step read
template <int M, bool MASS, int KC>
__device__ __forceinline__ void mt_ldb(const double* __restrict__ tiles, double (&b)[MtDims<M>::RT], const int (&dir)[2],
                                       const int (&trn)[2]) {
    constexpr int RT = MtDims<M>::RT, T = KC / 2, e = KC % 2;
    static_for<RT>([&](auto tc) {
        constexpr int t = decltype(tc)::value;
        if constexpr (!MASS || mt_face_tile(M, T, t)) {
            constexpr int hi = T >= t ? T : t, lo = T >= t ? t : T;
            constexpr int tl = MASS ? mt_mass_idx(M, hi, lo) : hi * (hi + 1) / 2 + lo;
            b[t] = tiles[tl * 64 + (T >= t ? dir[e] : trn[e])];
        }
    });
}

#ifndef MT_AHEAD
#define MT_AHEAD 3  // B fragments are loaded this many k-steps ahead of their MMAs (1: 0.595, 2: 0.592, 3: 0.589 ms/step)
#endif
template <int M, bool MASS, int KC>
__device__ __forceinline__ void mt_kstep(const double* __restrict__ tiles, const double (&x)[MtDims<M>::RT][2],
                                         double (&acc)[MtDims<M>::RT][2], double (&bb)[MT_AHEAD + 1][MtDims<M>::RT],
                                         const int (&dir)[2], const int (&trn)[2]) {
    constexpr int RT = MtDims<M>::RT, T = KC / 2, e = KC % 2, NB = MT_AHEAD + 1;
    if constexpr (KC + MT_AHEAD < 2 * RT) mt_ldb<M, MASS, KC + MT_AHEAD>(tiles, bb[(KC + MT_AHEAD) % NB], dir, trn);
    const double a = x[T][e];
    static_for<RT>([&](auto tc) {
        constexpr int t = decltype(tc)::value;
        if constexpr (!MASS || mt_face_tile(M, T, t)) dmma8x8x4(acc[t], a, bb[KC % NB][t]);
    });
    if constexpr (KC + 1 < 2 * RT) mt_kstep<M, MASS, KC + 1>(tiles, x, acc, bb, dir, trn);
}

// acc^T = x^T B over all row tiles; x, acc in accumulator-fragment layout (see the header comment).
// MASS: B = block-diagonal interface mass, only the tiles that meet a face block.  RT independent
// accumulator chains; every tile offset is an immediate.  The B fragments of k-step kc + 1 are loaded
// before the MMAs of k-step kc are issued.
template <int M, bool MASS>
__device__ __forceinline__ void mt_gemm(const double* __restrict__ tiles, const double (&x)[MtDims<M>::RT][2],
                                        double (&acc)[MtDims<M>::RT][2], const int (&dir)[2], const int (&trn)[2]) {
    constexpr int RT = MtDims<M>::RT;
#pragma unroll
    for (int t = 0; t < RT; ++t) acc[t][0] = acc[t][1] = 0.0;
    double bb[MT_AHEAD + 1][RT];
    static_for<MT_AHEAD>([&](auto kc) { mt_ldb<M, MASS, decltype(kc)::value>(tiles, bb[decltype(kc)::value], dir, trn); });
    mt_kstep<M, MASS, 0>(tiles, x, acc, bb, dir, trn);
}

template <int M>
__device__ __forceinline__ void mt_compute(const MtParams& p, const double* ring, uint64_t* full, uint64_t* empty,
                                           uint64_t* stepdone, const int* ssub, const int* s_id, const int* s_nb, int ns,
                                           int team, int w, int lane, double* stash) {
    using D = MtDims<M>;
    constexpr int S = D::S, W = D::W, RT = D::RT, WP = D::WP, SB = D::SB, STG = D::STG;
    const int L = p.L, NST = p.nst;
    const long long KS = (long long)L * SB;
    const int g = lane >> 2, c = lane & 3;
    const int q = 8 * w + g;              // this lane's shot
    const int lo = q * WP + 2 * c;        // offset of (shot q, row 2c) in a state block
    int dir[2], trn[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        dir[e] = mt_pos(2 * c + e, g);
        trn[e] = mt_pos(g, 2 * c + e);
    }
    // ring cursor (same item sequence in every compute warp and in the producer)
    int st = 0;
    uint32_t ph = 0;
    auto acquire = [&](int o) -> const double* {
        int s2 = st + o;
        uint32_t p2 = ph;
        if (s2 >= NST) {
            s2 -= NST;
            p2 ^= 1;
        }
        mbar_wait(&full[s2], p2);
        return ring + (size_t)s2 * STG;
    };
    auto release = [&]() {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == NST) {
            st = 0;
            ph ^= 1;
        }
    };
    auto load_slice = [&](const double* blk, double (&v)[RT][2]) {
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const double2 d = *reinterpret_cast<const double2*>(blk + lo + 8 * t);
            v[t][0] = d.x;
            v[t][1] = d.y;
        }
    };
    auto store_slice = [&](double* blk, const double (&v)[RT][2]) {
#pragma unroll
        for (int t = 0; t < RT; ++t)
            *reinterpret_cast<double2*>(blk + lo + 8 * t) = make_double2(v[t][0], v[t][1]);
    };
    // warp-private scratch for the two state slices a layer needs again after its products
    // (U_j for the leapfrog, U_{j+1} as the next layer's U_j): kept out of registers during the GEMMs
    double2* stw = reinterpret_cast<double2*>(stash) + (size_t)w * (3 * RT * 32) + lane;
    auto stash_put = [&](int slot, const double (&v)[RT][2]) {
#pragma unroll
        for (int t = 0; t < RT; ++t) stw[(slot * RT + t) * 32] = make_double2(v[t][0], v[t][1]);
    };
    const double dt2 = p.dt2;
    const int barT = 1 + (int)(threadIdx.x >= (MT_NCW + 1) * 32);  // named barrier of the team's compute warps
    const int my_src = ssub[q];           // source subdomain of this lane's shot
    const double* svec = my_src >= 0 ? p.shot_vec + p.shot_voff[q] : nullptr;

    // ---- layer 0 of one subdomain for the step whose fluxes are in fxb: T = F_0 + neighbour's F_0 on
    // shared faces, acc_0 = mass T (sparse tile GEMM) or the stored H_0 F_0 rows on outer faces, source,
    // leapfrog into ub (the buffer whose layer-0 slot still holds the older level); the new U_0 stays
    // in v.  Ring items: mass tiles, U_0 (newer level), U_0 (older level).
    auto layer0 = [&](int sl, const double* fxb, double fqv, double* ub, double& sqv, double (&v)[RT][2]) {
        const int s = s_id[sl];
        const bool mine = my_src == s;
        double x[RT][2], a1[RT][2], acc[RT][2];
        {
            // face values (own + neighbour flux on shared faces, acc_0 on outer faces; a row takes
            // exactly one of the two): scattered L2 reads
            const double* fo = fxb + (size_t)s * SB + lo;
            const double* ao = p.acc1 + (size_t)s * SB + lo;
#pragma unroll
            for (int t = 0; t < RT; ++t)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int row = 8 * t + 2 * c + e;
                    x[t][e] = 0.0;
                    a1[t][e] = 0.0;
                    if (row < W) {
                        const int f = row / M, nb = s_nb[sl * 6 + f];
                        if (nb >= 0)
                            x[t][e] = __dadd_rn(__ldcg(fo + 8 * t + e),
                                                __ldcg(fxb + (size_t)nb * SB + q * WP + (f ^ 1) * M + row % M));
                        else
                            a1[t][e] = __ldcg(ao + 8 * t + e);
                    }
                }
        }
        mt_gemm<M, true>(acquire(0), x, acc, dir, trn);
        const double* u0 = acquire(1);
        const double* uo = acquire(2);
        double* un = ub + (size_t)s * KS;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
            const double2 u = *reinterpret_cast<const double2*>(u0 + lo + 8 * t);
            const double2 o = *reinterpret_cast<const double2*>(uo + lo + 8 * t);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = 8 * t + 2 * c + e;
                double tot = __dadd_rn(acc[t][e], a1[t][e]);  // one of the two is zero
                if (mine && row < W) tot = __dadd_rn(tot, __dmul_rn(svec[row], fqv));
                v[t][e] = fma(dt2, tot, fma(2.0, e ? u.y : u.x, e ? -o.y : -o.x));
                sqv = fma(v[t][e], v[t][e], sqv);
            }
            *reinterpret_cast<double2*>(un + lo + 8 * t) = make_double2(v[t][0], v[t][1]);
        }
        release();  // mass tiles
        release();  // U_0, newer level
        release();  // U_0, older level
    };
    // per-shot |U|^2 partial of this team (the 4 lanes of a shot hold its rows); slot 0: layers >= 1
    // of step kz + 1, slot 1: its layer 0 (computed one sweep later)
    auto put_norm = [&](int kz, int slot, double sqv) {
        sqv += __shfl_xor_sync(0xffffffffu, sqv, 1);
        sqv += __shfl_xor_sync(0xffffffffu, sqv, 2);
        if (c == 0) p.norm_part[(((size_t)kz * 2 + slot) * p.n_team + team) * S + q] = sqv;
    };
    // probes: rows of the completed state after step kdone (thread = shot x every 4th probe); the
    // caller has passed a team barrier after the last write of that state
    auto record = [&](int kdone, const double* Ub) {
        if (kdone % p.record_every != 0 || !p.rows) return;
        const long long rec = kdone / p.record_every - 1;
        const int pq0 = w, qs = lane;  // thread (w, lane): shot lane, probes w, w+4, ...
        for (int sl = 0; sl < ns; ++sl) {
            const int s = s_id[sl];
            const double* us = Ub + (size_t)s * KS + (size_t)qs * WP;
            for (int pq = p.prb_ptr[s] + pq0; pq < p.prb_ptr[s + 1]; pq += MT_NCW) {
                const int pid = p.prb_ids[pq];
                const int tap = p.prb_tap[pid];
                double val;
                if (tap >= 0) {
                    val = us[(size_t)(tap / W) * SB + tap % W];
                } else {
                    const double* wv = p.prb_w + p.prb_woff[pid];
                    val = 0.0;
                    for (int j = 0; j < L; ++j)
                        for (int r = 0; r < W; ++r) val = fma(wv[j * W + r], us[(size_t)j * SB + r], val);
                }
                p.rows[(rec * S + qs) * p.n_probe + pid] = val;  // [rec][shot][probe]
            }
        }
    };

    for (int k = 1; k <= p.n_steps; ++k) {
        const int par = k & 1;
        const int cb = (k - 1) & 1;
        double* Un = cb ? p.U0 : p.U1;  // U^{k-2} -> U^k (layers >= 1 in this sweep, layer 0 one sweep later)
        double* Uc = cb ? p.U1 : p.U0;  // U^{k-1}; its layer 0 is completed in this sweep
        double* fx = p.flux + (size_t)par * p.n_sub * SB;
        const double* fxp = p.flux + (size_t)(par ^ 1) * p.n_sub * SB;  // F_0 of step k-1
        const int kk = k - 1;
        const double fq = my_src >= 0 ? p.ftab[(size_t)q * p.ftab_stride + kk] : 0.0;
        const double fqp = (my_src >= 0 && k >= 2) ? p.ftab[(size_t)q * p.ftab_stride + kk - 1] : 0.0;
        double sq = 0.0, sq0 = 0.0;

        // ---- sweep: per subdomain the deferred layer 0 of step k-1, then the layers of step k, in registers
        for (int sl = 0; sl < ns; ++sl) {
            const int s = s_id[sl];
            const bool mine = my_src == s;
            double x[RT][2], acc[RT][2];
            int cur = 0;  // stash slot of U_j (slot 2: the previous layer's flux F_{j-1})
            if (k == 1) {
                load_slice(acquire(0), x);  // U_0 of the start state
                release();
            } else {
                layer0(sl, fxp, fqp, Uc, sq0, x);  // U_0^{k-1}: all neighbours published F_0^{k-1} before the barrier
            }
            {
                double ua[RT][2];
                load_slice(acquire(0), ua);  // U_1
                release();
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    x[t][0] = ua[t][0] - x[t][0];
                    x[t][1] = ua[t][1] - x[t][1];
                }
                stash_put(cur, ua);
            }
            {
                double fp[RT][2];
                mt_gemm<M, false>(acquire(0), x, fp, dir, trn);  // F_0
                release();
                store_slice(fx + (size_t)s * SB, fp);
                stash_put(2, fp);
                const bool interior = (s_nb[sl * 6] | s_nb[sl * 6 + 1] | s_nb[sl * 6 + 2] | s_nb[sl * 6 + 3] |
                                       s_nb[sl * 6 + 4] | s_nb[sl * 6 + 5]) >= 0;
                if (!interior) {  // acc_0 = H_0 F_0: only outer-face rows are read back
                    mt_gemm<M, false>(acquire(0), fp, acc, dir, trn);
                    release();
                    store_slice(p.acc1 + (size_t)s * SB, acc);
                }
            }
            for (int j = 1; j < L; ++j) {
                {
                    double ub[RT][2];
                    if (j + 1 < L) {
                        load_slice(acquire(0), ub);  // U_{j+1}
                        release();
                    } else {
#pragma unroll
                        for (int t = 0; t < RT; ++t) ub[t][0] = ub[t][1] = 0.0;
                    }
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const double2 a = stw[(cur * RT + t) * 32];  // U_j
                        x[t][0] = ub[t][0] - a.x;
                        x[t][1] = ub[t][1] - a.y;
                    }
                    stash_put(cur ^ 1, ub);
                }
                mt_gemm<M, false>(acquire(0), x, acc, dir, trn);  // F_j
                release();
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const double2 f = stw[(2 * RT + t) * 32];  // F_{j-1}
                    x[t][0] = acc[t][0] - f.x;
                    x[t][1] = acc[t][1] - f.y;
                }
                stash_put(2, acc);
                mt_gemm<M, false>(acquire(0), x, acc, dir, trn);  // A_j
                release();
                const double* uo = acquire(0);  // Uprev_j
                double* un = Un + (size_t)s * KS + (size_t)j * SB;
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const double2 o = *reinterpret_cast<const double2*>(uo + lo + 8 * t);
                    const double2 a = stw[(cur * RT + t) * 32];  // U_j
                    double v[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        double tot = acc[t][e];
                        const int row = 8 * t + 2 * c + e;
                        if (mine && row < W) tot = __dadd_rn(tot, __dmul_rn(svec[(long long)j * W + row], fq));
                        v[e] = fma(dt2, tot, fma(2.0, e ? a.y : a.x, e ? -o.y : -o.x));
                        sq = fma(v[e], v[e], sq);
                    }
                    *reinterpret_cast<double2*>(un + lo + 8 * t) = make_double2(v[0], v[1]);
                }
                release();
                cur ^= 1;
            }
        }
        // ---------------- grid-wide step barrier ------------------------------------------
        // (bar.sync orders the team's face-buffer writes before lane 0's release store: cumulativity.)
        // Layer 0 of step k reads only face neighbours' buffers; the wait is for every team (the
        // grid-wide barrier per step), which measured the same step time as neighbour-only flags.
        asm volatile("bar.sync %0, %1;" ::"r"(barT), "r"(MT_NCW * 32) : "memory");
        if (w == 0 && lane == 0) st_release(p.flags + team, (unsigned int)k);
        // while the other teams finish: norms, and the probes of step k-1 (its layer 0 was written by this
        // team's warps before the barrier above)
        put_norm(kk, 0, sq);
        if (k >= 2) {
            put_norm(kk - 1, 1, sq0);
            record(k - 1, Uc);
        }
        if (w == 0) {
            for (int i = lane; i < p.n_team; i += 32)
                while (ld_acquire(p.flags + i) < (unsigned int)k) {
                }
            __syncwarp();
        }
        asm volatile("bar.sync %0, %1;" ::"r"(barT), "r"(MT_NCW * 32) : "memory");
        // this step's state writes feed the next step's bulk-copy reads (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(stepdone);
    }
    // ---------------- epilogue: layer 0 of the last step ------------------------------------
    {
        const int k = p.n_steps;
        double* Un = ((k - 1) & 1) ? p.U0 : p.U1;
        const double* fx = p.flux + (size_t)(k & 1) * p.n_sub * SB;
        const double fq = my_src >= 0 ? p.ftab[(size_t)q * p.ftab_stride + k - 1] : 0.0;
        double sq0 = 0.0;
        for (int sl = 0; sl < ns; ++sl) {
            double v[RT][2];
            layer0(sl, fx, fq, Un, sq0, v);
        }
        put_norm(k - 1, 1, sq0);
        asm volatile("bar.sync %0, %1;" ::"r"(barT), "r"(MT_NCW * 32) : "memory");  // the team's U rows are written
        record(k, Un);
    }
}

template <int M>
__global__ void __launch_bounds__(2 * (MT_NCW + 1) * 32, 1) k_step_mt(const MtParams p) {
    using D = MtDims<M>;
    constexpr int S = D::S, TB = D::TB, SB = D::SB, STG = D::STG, NMT = D::NMT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // a CTA hosts two independent teams (5 warps each: 4 compute + 1 producer) with their own rings,
    // subdomain ranges and step flags: two sweeps in flight per SM, two compute warps per SMSP
    const int tw = threadIdx.x / ((MT_NCW + 1) * 32);
    const int team = 2 * blockIdx.x + tw;
    if (team >= p.n_team) return;
    const int tid = threadIdx.x - tw * (MT_NCW + 1) * 32;
    const int warp = tid >> 5, lane = tid & 31;
    const int L = p.L, NST = p.nst;
    const long long KS = (long long)L * SB;
    double* ring = reinterpret_cast<double*>(smem_raw + (size_t)tw * p.team_smem);  // [NST][STG]
    double* stash = ring + (size_t)NST * STG;  // [MT_NCW][3][RT][32] double2, warp-private
    uint64_t* full = reinterpret_cast<uint64_t*>(stash + (size_t)MT_NCW * 3 * D::RT * 32 * 2);
    uint64_t* empty = full + NST;
    uint64_t* stepdone = empty + NST;
    int* ssub = reinterpret_cast<int*>(stepdone + 1);
    int* s_id = ssub + S;        // [ns] the team's subdomains
    int* s_nb = s_id + p.nsmax;  // [ns][6] their face neighbours

    for (int i = tid; i < S; i += (MT_NCW + 1) * 32) ssub[i] = p.shot_sub[i];
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], MT_NCW);
        }
        mbar_init(stepdone, MT_NCW);
        fence_mbar_init();
    }
    const int s0 = p.cta_sub_ptr[team], s1 = p.cta_sub_ptr[team + 1];
    const int ns = s1 - s0;
    for (int i = tid; i < ns; i += (MT_NCW + 1) * 32) s_id[i] = p.team_subs[s0 + i];
    for (int i = tid; i < ns * 6; i += (MT_NCW + 1) * 32) s_nb[i] = p.nbr[p.team_subs[s0 + i / 6] * 6 + i % 6];
    asm volatile("bar.sync %0, %1;" ::"r"(3 + tw), "r"((MT_NCW + 1) * 32) : "memory");

    if (warp < MT_NCW) {
        mt_compute<M>(p, ring, full, empty, stepdone, ssub, s_id, s_nb, ns, team, warp, lane, stash);
        return;
    }
    // ======== producer: one lane streams every item in consumption order ========
    // Interior subdomains never read acc_0 (only outer-face rows do), so their Gamma-hat_0
    // block is not streamed.  State items of step k wait for the compute warps' step k-1.
    if (lane != 0) return;
    const uint64_t pol = l2_policy_evict_first();
    constexpr uint32_t cbytes = (uint32_t)TB * 8u, sbytes = (uint32_t)SB * 8u, mbytes = (uint32_t)NMT * 512u;
    int st = 0;
    uint32_t ph = 0;
    auto issue = [&](const double* src, uint32_t bytes) {
        mbar_wait(&empty[st], ph ^ 1);
        // The compute warps read this stage through the generic proxy; the bulk copy writes it through
        // the async proxy.  The proxy fence between the acquire above and the copy is REQUIRED: without it
        // the kernel was not repeatable run to run at full size (a refill could overtake reads of the
        // stage still in flight, config 4, has the history of that bug).
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[st], bytes);
        bulk_g2s(ring + (size_t)st * STG, src, bytes, &full[st], pol);
        if (++st == NST) {
            st = 0;
            ph ^= 1;
        }
    };
    for (int k = 0; k < p.n_steps; ++k) {
        if (k > 0) mbar_wait(stepdone, (uint32_t)((k - 1) & 1));
        const double* cur = (k & 1) ? p.U1 : p.U0;
        const double* prv = (k & 1) ? p.U0 : p.U1;
        for (int sl = 0; sl < ns; ++sl) {
            const bool interior = (s_nb[sl * 6] | s_nb[sl * 6 + 1] | s_nb[sl * 6 + 2] | s_nb[sl * 6 + 3] |
                                   s_nb[sl * 6 + 4] | s_nb[sl * 6 + 5]) >= 0;
            const double* uc = cur + (long long)s_id[sl] * KS;
            const double* up = prv + (long long)s_id[sl] * KS;
            const double* cf = p.tcoef + (long long)s_id[sl] * 2 * L * TB;
            if (k == 0) {
                issue(uc, sbytes);
            } else {  // deferred layer 0 of the previous step: its U_0 levels are prv (newer) and cur's stale slot
                issue(p.mtiles + (size_t)s_id[sl] * NMT * 64, mbytes);
                issue(up, sbytes);
                issue(uc, sbytes);
            }
            issue(uc + SB, sbytes);
            issue(cf, cbytes);
            if (!interior) issue(cf + TB, cbytes);
            for (int j = 1; j < L; ++j) {
                if (j + 1 < L) issue(uc + (long long)(j + 1) * SB, sbytes);
                issue(cf + (long long)(2 * j) * TB, cbytes);
                issue(cf + (long long)(2 * j + 1) * TB, cbytes);
                issue(up + (long long)j * SB, sbytes);
            }
        }
    }
    // epilogue: layer 0 of the last step (its newer U_0 level was written during that step's sweep)
    {
        const int k = p.n_steps - 1;
        mbar_wait(stepdone, (uint32_t)(k & 1));
        const double* cur = (k & 1) ? p.U1 : p.U0;
        const double* prv = (k & 1) ? p.U0 : p.U1;
        for (int sl = 0; sl < ns; ++sl) {
            issue(p.mtiles + (size_t)s_id[sl] * NMT * 64, mbytes);
            issue(cur + (long long)s_id[sl] * KS, sbytes);
            issue(prv + (long long)s_id[sl] * KS, sbytes);
        }
    }
}

static const void* mt_kernel(int m) {
    static const void* const tab[10] = {nullptr,
                                        (const void*)k_step_mt<1>,
                                        (const void*)k_step_mt<2>,
                                        (const void*)k_step_mt<3>,
                                        (const void*)k_step_mt<4>,
                                        (const void*)k_step_mt<5>,
                                        (const void*)k_step_mt<6>,
                                        (const void*)k_step_mt<7>,
                                        (const void*)k_step_mt<8>,
                                        (const void*)k_step_mt<9>};
    return (m >= 1 && m <= 9) ? tab[m] : nullptr;
}

struct MtShape {
    int W, RT, WP, TB, SB, STG, NMT;
};

static MtShape mt_shape(int m) {
    MtShape d;
    d.W = 6 * m;
    d.RT = (d.W + 7) / 8;
    d.WP = 8 * d.RT;
    d.TB = d.RT * (d.RT + 1) / 2 * 64;
    d.SB = 32 * d.WP;
    d.STG = std::max(d.TB, d.SB);
    d.NMT = mt_mass_count(m);
    return d;
}

static size_t mt_smem_bytes(const MtShape& d, int nst, int nsmax) {
    const size_t b = (size_t)nst * d.STG * 8 + (size_t)MT_NCW * 3 * d.RT * 32 * 16 + (2 * (size_t)nst + 1) * 8 +
                     4 * (32 + 7 * (size_t)nsmax);
    return (b + 127) & ~(size_t)127;  // one team
}

// shots start from rest (u0 = v0 = 0): U_curr = 0, U_prev = ((0.5 dt) dt) (vec_q f_q(0))  (stepper.py:347-353)
__global__ void k_ms_init(double* U0, double* U1, long long total, int S, int W, int WP, int L, const int* shot_sub,
                          const double* shot_vec, const long long* shot_voff, const double* f0, double half) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i % WP);
        long long rest = i / WP;
        const int q = (int)(rest % S);
        rest /= S;
        const int j = (int)(rest % L);
        const long long s = rest / L;
        U0[i] = 0.0;
        double v = 0.0;
        if (r < W && shot_sub[q] == s) v = __dmul_rn(half, __dmul_rn(shot_vec[shot_voff[q] + (long long)j * W + r], f0[q]));
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

// one shot of the [sub][layer][shot][WP] state as the reference's concatenated [sub][L*W] vector
__global__ void k_mt_gather(const double* __restrict__ U, long long total, int q, int S, int W, int WP,
                            double* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i % W);
        const long long sj = i / W;  // s * L + j
        out[i] = U[(sj * S + q) * WP + r];
    }
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
    if (h->L < 2) return fail(SFW_ECONFIG, "multi-shot stepping needs at least 2 layers", errbuf, errlen);
    const void* kfn = mt_kernel(h->m);
    if (!kfn) return fail(SFW_ECONFIG, "multi-shot stepping supports 1 <= modes per face <= 9", errbuf, errlen);
    const int S = n_shots, L = h->L, n = h->n_sub;
    const MtShape d = mt_shape(h->m);
    h->TB = d.TB;
    h->n_shots = S;
    int rc = 0;
    if (!h->tcoef) {
        if ((rc = dalloc(&h->tcoef, (size_t)h->n_blocks * d.TB, errbuf, errlen))) return rc;
        k_tilepack<<<(unsigned)h->n_blocks, 256, 0, h->stream>>>(h->coef, h->BS, h->m, d.RT, d.TB, h->tcoef,
                                                                 h->n_blocks);
    }
    if (!h->mmass) {
        if ((rc = dalloc(&h->mmass, (size_t)n * d.NMT * 64, errbuf, errlen))) return rc;
        k_mt_masstiles<<<(unsigned)n, 64, 0, h->stream>>>(h->mass, h->mass_idx, n, h->m, d.RT, d.NMT, h->mmass);
    }
    const size_t st = (size_t)n * L * d.SB;
    for (int b = 0; b < 2; ++b)
        if (!h->UM[b] && (rc = dalloc(&h->UM[b], st, errbuf, errlen))) return rc;
    if (!h->mfb && (rc = dalloc(&h->mfb, (size_t)2 * n * d.SB, errbuf, errlen))) return rc;
    if (!h->macc1 && (rc = dalloc(&h->macc1, (size_t)n * d.SB, errbuf, errlen))) return rc;
    std::vector<long long> voff(S);
    long long vt = 0;
    for (int q = 0; q < S; ++q) {
        const int s = shot_sub[q];
        if (s < -1 || s >= n) return fail(SFW_ECONFIG, "shot source subdomain has no model", errbuf, errlen);
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
    if (!h->mt_grid) {
        // work decomposition: two teams per SM, each a contiguous subdomain range
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        int G = std::min(2 * nsm, n);
        if (const char* e = getenv("SFW_STEP_MAXGRID")) G = std::max(1, std::min(G, atoi(e)));  // test hook
        // A step ends at a grid-wide barrier, so the most loaded team sets its length.  Cost of a
        // subdomain: 2L-1 block products, one more (Gamma-hat_0) on the domain boundary, plus the
        // face pass.  Longest-processing-time assignment (costliest first, to the least loaded team;
        // ties to the lower team so that runs of neighbours stay together), ascending within a team.
        std::vector<int> order(n), cost(n);
        for (int sdx = 0; sdx < n; ++sdx) {
            bool interior = true;
            for (int f = 0; f < 6; ++f) interior = interior && h->nbr_h[6 * sdx + f] >= 0;
            cost[sdx] = 10 * (2 * L - 1) + 6 + (interior ? 0 : 10);
            order[sdx] = sdx;
        }
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
        std::vector<long long> load(G, 0);
        std::vector<std::vector<int>> mine(G);
        for (int sdx : order) {
            int best = 0;
            for (int b = 1; b < G; ++b)
                if (load[b] < load[best]) best = b;
            load[best] += cost[sdx];
            mine[best].push_back(sdx);
        }
        std::vector<int> cta_ptr(G + 1, 0), subs;
        int nsmax = 0;
        for (int b = 0; b < G; ++b) {
            std::sort(mine[b].begin(), mine[b].end());
            subs.insert(subs.end(), mine[b].begin(), mine[b].end());
            cta_ptr[b + 1] = (int)subs.size();
            nsmax = std::max(nsmax, (int)mine[b].size());
        }
        if ((rc = upload(&h->mt_cta_ptr, cta_ptr, errbuf, errlen))) return rc;
        if ((rc = upload(&h->mt_ncta, subs, errbuf, errlen))) return rc;  // the teams' subdomain lists
        h->mt_nsmax = nsmax;
        if ((rc = dalloc(&h->mt_flags, (size_t)G, errbuf, errlen))) return rc;
        // ring depth: two teams share the 227 KB of a CTA
        int nst = 12;
        while (nst > 4 && 2 * mt_smem_bytes(d, nst, nsmax) > 226 * 1024) --nst;
        const size_t smem = 2 * mt_smem_bytes(d, nst, nsmax);
        if (smem > 227 * 1024)
            return fail(SFW_ECONFIG, "multi-shot stepping: too many subdomains per CTA for shared memory", errbuf,
                        errlen);
        SFW_CUDA_TRY(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        SFW_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, 2 * (MT_NCW + 1) * 32, smem));
        if (per_sm * nsm < (G + 1) / 2) {
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, kfn);
            return fail(SFW_ECONFIG,
                        "multi-shot stepping: the persistent grid is not co-resident (registers " +
                            std::to_string(fa.numRegs) + ", max threads " + std::to_string(fa.maxThreadsPerBlock) +
                            ", shared " + std::to_string(smem) + " B, CTAs per SM " + std::to_string(per_sm) + ")",
                        errbuf, errlen);
        }
        h->mt_team_smem = (int)mt_smem_bytes(d, nst, nsmax);
        h->mt_nst = nst;
        h->shot_smem2 = (int)smem;
        h->mt_grid = G;
    }
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    return 0;
}

// Run n_steps from rest for all shots.  profile: HOST [S][n_steps] f_q(t_k), t_k = k dt;
// profile0: HOST [S] f_q(0).  rows_out: HOST [n_steps/record_every][S][n_probe] (or NULL);
// norms_out: HOST [n_steps][S] (or NULL); *kernel_ms: CUDA-event time of the launch.
extern "C" int sfw_shots_run(sfw_stepper* h, int n_steps, int record_every, const double* profile0,
                             const double* profile, double* rows_out, double* norms_out, float* kernel_ms,
                             char* errbuf, int errlen) {
    if (!h->n_shots) return fail(SFW_ECONFIG, "call sfw_shots_setup first", errbuf, errlen);
    if (n_steps <= 0) return 0;
    if (record_every < 1) return fail(SFW_ECONFIG, "record_every must be >= 1", errbuf, errlen);
    const int S = h->n_shots, L = h->L;
    const MtShape d = mt_shape(h->m);
    int rc = ms_ensure(&h->shot_ftab, &h->shot_ftab_cap, (long long)S * n_steps + S, errbuf, errlen);
    if (rc) return rc;
    SFW_CUDA_TRY(cudaMemcpyAsync(h->shot_ftab, profile, (size_t)S * n_steps * 8, cudaMemcpyHostToDevice, h->stream));
    SFW_CUDA_TRY(cudaMemcpyAsync(h->shot_ftab + (size_t)S * n_steps, profile0, (size_t)S * 8, cudaMemcpyHostToDevice,
                                 h->stream));
    const long long nrec = n_steps / record_every;
    if ((rc = ms_ensure(&h->mrows, &h->mrows_cap, std::max(1LL, nrec * h->n_probe * S), errbuf, errlen))) return rc;
    const int nparts = 2 * h->mt_grid;  // |U|^2 partials per step: two per team (layers >= 1, layer 0)
    if ((rc = ms_ensure(&h->mnorm, &h->mnorm_cap, (long long)n_steps * nparts * S + (long long)n_steps * S, errbuf,
                        errlen)))
        return rc;
    const long long total = (long long)h->n_sub * L * d.SB;
    const double half = (0.5 * h->dt) * h->dt;
    k_ms_init<<<1184, 256, 0, h->stream>>>(h->UM[0], h->UM[1], total, S, d.W, d.WP, L, h->shot_sub, h->shot_vec,
                                           h->shot_voff, h->shot_ftab + (size_t)S * n_steps, half);
    SFW_CUDA_TRY(cudaMemsetAsync(h->mt_flags, 0, sizeof(unsigned int) * h->mt_grid, h->stream));
    MtParams p{};
    p.n_sub = h->n_sub;
    p.L = L;
    p.n_steps = n_steps;
    p.record_every = record_every;
    p.n_probe = h->n_probe;
    p.ftab_stride = n_steps;
    p.nst = h->mt_nst;
    p.n_team = h->mt_grid;
    p.team_smem = h->mt_team_smem;
    p.dt2 = h->dt * h->dt;
    p.tcoef = h->tcoef;
    p.mtiles = h->mmass;
    p.U0 = h->UM[0];
    p.U1 = h->UM[1];
    p.flux = h->mfb;
    p.acc1 = h->macc1;
    p.nbr = h->nbr;
    p.cta_sub_ptr = h->mt_cta_ptr;
    p.team_subs = h->mt_ncta;
    p.nsmax = h->mt_nsmax;
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
    p.flags = h->mt_flags;
    void* args[] = {&p};
    SFW_CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
    SFW_CUDA_TRY(cudaLaunchCooperativeKernel(mt_kernel(h->m), dim3((h->mt_grid + 1) / 2), dim3(2 * (MT_NCW + 1) * 32), args,
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
    const MtShape d = mt_shape(h->m);
    const long long total = (long long)h->n_sub * h->L * d.W;
    double* tmp = nullptr;
    int rc = dalloc(&tmp, (size_t)total, errbuf, errlen);
    if (rc) return rc;
    for (int lvl = 0; lvl < 2; ++lvl) {
        double* dst = lvl == 0 ? u_curr : u_prev;
        if (!dst) continue;
        const double* src = h->UM[lvl == 0 ? h->mcur : h->mcur ^ 1];
        k_mt_gather<<<592, 256, 0, h->stream>>>(src, total, q, h->n_shots, d.W, d.WP, tmp);
        cudaError_t e = cudaMemcpyAsync(dst, tmp, (size_t)total * 8, cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) {
            cudaFree(tmp);
            return SFW_ECUDA;
        }
    }
    cudaFree(tmp);
    return 0;
}

// algorithmic bytes / flops per step of the multi-shot launch (SURVEY 8d, S shots), and the
// bytes the kernel streams (tile-padded blocks, padded state rows, mass tiles, face buffer)
extern "C" int sfw_shots_traffic(sfw_stepper* h, double* alg_bytes, double* alg_flops, double* streamed) {
    const double w = h->W, S = h->n_shots ? h->n_shots : 32;
    const MtShape d = mt_shape(h->m);
    double b = 0, f = 0, s = 0;
    for (int i = 0; i < h->n_sub; ++i) {
        const double L = h->layers[i];
        b += 8.0 * ((2 * L - 1) * w * (w + 1) / 2 + 3 * L * w * S);
        f += S * (2.0 * (2 * L - 1) * w * w + 5 * L * w);
        s += 8.0 * ((2 * L - 1) * d.TB + d.NMT * 64 + (3 * L + 1) * (double)d.SB);
    }
    if (alg_bytes) *alg_bytes = b;
    if (alg_flops) *alg_flops = f;
    if (streamed) *streamed = s;
    return 0;
}
