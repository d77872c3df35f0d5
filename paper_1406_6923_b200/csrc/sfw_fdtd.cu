// Fine-grid leapfrog reference solver on the GPU (reference reference.py:26-157,
// operator grid.py:326-382 + 461-467).
//
// The reference integrates w_tt = A w + f(t) s on the undecomposed grid, with A = -C Lap_h C the
// link-weighted graph stiffness (mirror closure) as a scipy CSR matrix.  Here A is never stored:
// every thread rebuilds its row from c and the per-axis scales 1/h_d^2 in the reference's exact
// arithmetic --
//   off-diagonal (i, j):  (c_lo * c_hi) * s_d                      (grid.py:365-372)
//   diagonal:             0 + sum over links in the order d = x, y, z, lower end then upper end
//                         of (-c_i * c_i) * s_d                      (np.add.at, grid.py:373-374)
//   row product:          0 + sum of a_ij * w_j over the sorted columns x-, y-, z-, i, z+, y+, x+
//                         (scipy csr_matvec, no FMA)
// and the leapfrog / start / forcing in numpy's evaluation order (reference.py:117-135), so the GPU
// trajectory is the reference's bit for bit (tests/test_fdtd_gpu.py).
//
// Layout: C-order (x, y, z), z fastest; fp64 c, and two time levels ping-ponged in place (level
// k+1 overwrites level k-1 element-wise).  HBM sees u, c, u_prev read once and u_next written
// once -- 32 B per node-step, the kernel's roofline (HBM-bound: 13 flop per 32 B); see k_fdtd
// for the 2.5-D blocking that gets there.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "sfw_common.cuh"

namespace sfw {

struct FdParams {
    int nx, ny, nz;
    double s0, s1, s2;     // 1/h_d^2 exactly as the reference forms them
    const double* c;
    const double* u;       // current level (or the vector A is applied to)
    double* out;           // mode 0: previous level in, next level out; 1: start level; 2: -A u
    const double* vel;     // mode 1: initial velocity or null
    double dt, dt2, half;  // dt, dt*dt, (0.5*dt)*dt
    const double* damping; // mode 0: per-node factor or null
    int n_src;
    const long long* src_idx;
    const double* src_val;
    double f;              // source profile value of this step
    double* part;          // per-block partial sums: mode 0/1 |out|^2, mode 2 unused
    int n_rec;             // mode 0: receivers written by the kernel into rows (when rows != null)
    const long long* rec;
    double* rows;          // mode 0: this step's receiver row, or null
};

// 2.5-D blocking: a CTA owns a 32 (z) x 8 (y) column of XC consecutive x-planes.  The thread's
// own node of planes x-1, x, x+1 lives in registers (u and c), the current plane's y/z halo in
// shared memory, so HBM sees each u, c, u_prev once and L2 only the tile halos.  The row sum is
// formed in the reference's order (x-, y-, z-, diag, z+, y+, x+) whatever the operands' source.
constexpr int FD_XC = 16;

template <int MODE, bool INT>
__device__ __forceinline__ void fdtd_tile(const FdParams& p, double (&su)[10][34], double (&sc)[10][34],
                                          double* red) {
    const int tz = threadIdx.x, ty = threadIdx.y;
    const int z = blockIdx.x * 32 + tz, y = blockIdx.y * 8 + ty;
    const int x0 = blockIdx.z * FD_XC, x1 = min(p.nx, x0 + FD_XC);
    const int sx = p.ny * p.nz, sy = p.nz;  // 32-bit offsets: grids up to 2^31 nodes (checked at create)
    const bool in = INT || (z < p.nz && y < p.ny);
    const int col = y * p.nz + z;
    // does this CTA's column hold a source node?  (block-uniform; the per-node test runs only there)
    bool src_here = false;
    for (int q = 0; q < p.n_src; ++q) {
        const long long s = p.src_idx[q];
        const int sxq = (int)(s / sx), rem = (int)(s % sx), syq = rem / p.nz, szq = rem % p.nz;
        src_here |= sxq >= x0 && sxq < x1 && syq / 8 == (int)blockIdx.y && szq / 32 == (int)blockIdx.x;
    }
    // does this CTA's column hold a receiver that is recorded this step?  (block-uniform)
    bool rec_here = false;
    if (MODE == 0 && p.rows)
        for (int q = 0; q < p.n_rec; ++q) {
            const long long r = p.rec[q];
            const int rx = (int)(r / sx), rem = (int)(r % sx), ry = rem / p.nz, rz = rem % p.nz;
            rec_here |= rx >= x0 && rx < x1 && ry / 8 == (int)blockIdx.y && rz / 32 == (int)blockIdx.x;
        }
    // halo duty of this thread: row y-1 (ty == 0), row y+1 (ty == 7), column z-1 (tz == 0), z+1 (tz == 31)
    const int hy = (ty == 0 && (INT || y > 0)) ? -1 : (ty == 7 && (INT || y + 1 < p.ny)) ? 1 : 0;
    const int hz = (tz == 0 && (INT || z > 0)) ? -1 : (tz == 31 && (INT || z + 1 < p.nz)) ? 1 : 0;
    // software pipeline, two planes deep: centre (u, c) of x+1 and x+2, halos and u_prev of x+1
    auto ld = [&](const double* a, int i) { return __ldg(a + i); };
    double um = 0.0, uc = 0.0, up = 0.0, u2 = 0.0, cm = 0.0, cc = 0.0, cp = 0.0, c2 = 0.0;
    double hyu = 0.0, hyc = 0.0, hzu = 0.0, hzc = 0.0, prv = 0.0, vel = 0.0;
    if (in) {
        const int i0 = x0 * sx + col;
        if (INT || x0 > 0) {
            um = ld(p.u, i0 - sx);
            cm = ld(p.c, i0 - sx);
        }
        uc = ld(p.u, i0);
        cc = ld(p.c, i0);
        if (INT || x0 + 1 < p.nx) {
            up = ld(p.u, i0 + sx);
            cp = ld(p.c, i0 + sx);
        }
        if (hy) {
            hyu = ld(p.u, i0 + hy * sy);
            hyc = ld(p.c, i0 + hy * sy);
        }
        if (hz) {
            hzu = ld(p.u, i0 + hz);
            hzc = ld(p.c, i0 + hz);
        }
        if (MODE == 0) prv = p.out[i0];
        if (MODE == 1 && p.vel) vel = p.vel[i0];
    }
    double sq = 0.0;
    for (int x = x0; x < x1; ++x) {
        const int i = x * sx + col;
        // current plane into shared memory (centre + halo)
        su[ty + 1][tz + 1] = uc;
        sc[ty + 1][tz + 1] = cc;
        if (hy) {
            su[ty + 1 + hy][tz + 1] = hyu;
            sc[ty + 1 + hy][tz + 1] = hyc;
        }
        if (hz) {
            su[ty + 1][tz + 1 + hz] = hzu;
            sc[ty + 1][tz + 1 + hz] = hzc;
        }
        const double prev = prv, v0 = vel;
        // next loads: plane x+2 centre, plane x+1 halos and u_prev
        if (in) {
            if (INT || x + 2 < p.nx) {
                u2 = ld(p.u, i + 2 * sx);
                c2 = ld(p.c, i + 2 * sx);
            }
            if (x + 1 < x1) {
                if (hy) {
                    hyu = ld(p.u, i + sx + hy * sy);
                    hyc = ld(p.c, i + sx + hy * sy);
                }
                if (hz) {
                    hzu = ld(p.u, i + sx + hz);
                    hzc = ld(p.c, i + sx + hz);
                }
                if (MODE == 0) prv = p.out[i + sx];
                if (MODE == 1 && p.vel) vel = p.vel[i + sx];
            }
        }
        __syncthreads();
        if (in) {
            const double ci = cc, ui = uc;
            const double cn = __dmul_rn(-ci, ci);
            double diag = 0.0;  // np.add.at order: x lower/upper end, y, z
            if (INT || p.nx > 1) {
                if (INT || x + 1 < p.nx) diag = __dadd_rn(diag, __dmul_rn(cn, p.s0));
                if (INT || x > 0) diag = __dadd_rn(diag, __dmul_rn(cn, p.s0));
            }
            if (INT || p.ny > 1) {
                if (INT || y + 1 < p.ny) diag = __dadd_rn(diag, __dmul_rn(cn, p.s1));
                if (INT || y > 0) diag = __dadd_rn(diag, __dmul_rn(cn, p.s1));
            }
            if (INT || p.nz > 1) {
                if (INT || z + 1 < p.nz) diag = __dadd_rn(diag, __dmul_rn(cn, p.s2));
                if (INT || z > 0) diag = __dadd_rn(diag, __dmul_rn(cn, p.s2));
            }
            double acc = 0.0;
            auto term = [&](double cj, double uj, double s) {
                acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(cj, ci), s), uj));
            };
            if (INT || x > 0) term(cm, um, p.s0);
            if (INT || y > 0) term(sc[ty][tz + 1], su[ty][tz + 1], p.s1);
            if (INT || z > 0) term(sc[ty + 1][tz], su[ty + 1][tz], p.s2);
            acc = __dadd_rn(acc, __dmul_rn(diag, ui));
            if (INT || z + 1 < p.nz) term(sc[ty + 1][tz + 2], su[ty + 1][tz + 2], p.s2);
            if (INT || y + 1 < p.ny) term(sc[ty + 2][tz + 1], su[ty + 2][tz + 1], p.s1);
            if (INT || x + 1 < p.nx) term(cp, up, p.s0);
            if (MODE == 2) {
                p.out[i] = -acc;
            } else {
                if (src_here)  // acc + f(t) * source_vec (reference.py:117-121)
                    for (int q = 0; q < p.n_src; ++q)
                        if (p.src_idx[q] == i) acc = __dadd_rn(acc, __dmul_rn(p.f, p.src_val[q]));
                double v;
                if (MODE == 0) {  // 2 u - u_prev + (dt*dt) acc   (reference.py:131)
                    v = __dadd_rn(__dsub_rn(__dmul_rn(2.0, ui), prev), __dmul_rn(p.dt2, acc));
                    if (p.damping) v = __dmul_rn(v, p.damping[i]);
                } else {          // u - dt v + (0.5 dt dt) acc   (reference.py:124)
                    v = __dadd_rn(__dsub_rn(ui, __dmul_rn(p.dt, v0)), __dmul_rn(p.half, acc));
                }
                p.out[i] = v;
                sq = fma(v, v, sq);
                if (MODE == 0 && rec_here)  // receiver rows straight from the new level
                    for (int q = 0; q < p.n_rec; ++q)
                        if (p.rec[q] == i) p.rows[q] = v;
            }
        }
        __syncthreads();
        um = uc;
        cm = cc;
        uc = up;
        cc = cp;
        up = u2;
        cp = c2;
    }
    if (MODE != 2) {  // fixed-order block partial of |out|^2 (deterministic)
        const double w = warp_sum(sq);
        if (tz == 0) red[ty] = w;
        __syncthreads();
        if (ty == 0 && tz == 0) {
            double t = 0.0;
            for (int k = 0; k < 8; ++k) t += red[k];
            p.part[((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
        }
    }
}


template <int MODE>
__global__ void __launch_bounds__(256) k_fdtd(const FdParams p) {
    __shared__ double su[10][34], sc[10][34];
    __shared__ double red[8];
    // block-uniform: a tile that touches no face of the grid takes the branch-free path (every
    // neighbour exists, so the same multiplies and adds run in the same order: bit-identical)
    const int z0 = blockIdx.x * 32, y0 = blockIdx.y * 8, x0 = blockIdx.z * FD_XC;
    const bool interior = z0 > 0 && z0 + 32 < p.nz && y0 > 0 && y0 + 8 < p.ny && x0 > 0 && x0 + FD_XC + 1 < p.nx;
    if (interior)
        fdtd_tile<MODE, true>(p, su, sc, red);
    else
        fdtd_tile<MODE, false>(p, su, sc, red);
}

// one block per step: the fixed-order sum of that step's block partials (the order k_fd_finish uses)
__global__ void k_fd_norms(const double* __restrict__ part, long long nparts, double* __restrict__ out) {
    __shared__ double red[32];
    const double* pk = part + (size_t)blockIdx.x * nparts;
    double t = 0.0;
    for (long long k = threadIdx.x; k < nparts; k += blockDim.x) t += pk[k];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        out[blockIdx.x] = s;
    }
}

// one block: fixed-order sum of the block partials -> out[slot]; gather of the receiver rows
__global__ void k_fd_finish(const double* __restrict__ part, long long nparts, double* __restrict__ out, int slot,
                            const double* __restrict__ u, const long long* __restrict__ rec, int n_rec,
                            double* __restrict__ rows) {
    __shared__ double red[32];
    double t = 0.0;
    for (long long k = threadIdx.x; k < nparts; k += blockDim.x) t += part[k];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        out[slot] = s;
    }
    if (rows)
        for (int r = threadIdx.x; r < n_rec; r += blockDim.x) rows[r] = u[rec[r]];
}

// power iteration pieces: partials of v.w and w.w, then v <- w / |w|
__global__ void k_fd_dots(const double* __restrict__ v, const double* __restrict__ w, long long n,
                          double* __restrict__ part) {
    double a = 0.0, b = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        a = fma(v[i], w[i], a);
        b = fma(w[i], w[i], b);
    }
    __shared__ double ra[32], rb[32];
    a = warp_sum(a);
    b = warp_sum(b);
    if ((threadIdx.x & 31) == 0) {
        ra[threadIdx.x >> 5] = a;
        rb[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sa = 0.0, sb = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            sa += ra[k];
            sb += rb[k];
        }
        part[2 * blockIdx.x] = sa;
        part[2 * blockIdx.x + 1] = sb;
    }
}

__global__ void k_fd_dots_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
    __shared__ double ra[32], rb[32];
    double a = 0.0, b = 0.0;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        a += part[2 * k];
        b += part[2 * k + 1];
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if ((threadIdx.x & 31) == 0) {
        ra[threadIdx.x >> 5] = a;
        rb[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sa = 0.0, sb = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            sa += ra[w];
            sb += rb[w];
        }
        out[0] = sa;
        out[1] = sb;
    }
}

__global__ void k_fd_scale(const double* __restrict__ w, double inv, long long n, double* __restrict__ v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] = w[i] / inv;
}

}  // namespace sfw

using namespace sfw;

struct sfw_fdtd {
    int nx = 0, ny = 0, nz = 0;
    long long n = 0;
    double s[3] = {0, 0, 0};
    double* c = nullptr;
    double* U[2] = {nullptr, nullptr};
    double* W = nullptr;      // scratch (apply / power iteration / velocity)
    double* part = nullptr;   // block partials
    double* acc = nullptr;    // device reduction results [>= 2]
    double* norms = nullptr;  // [cap] per-step |u|^2
    double* rows = nullptr;   // [cap_rows]
    long long norms_cap = 0, rows_cap = 0;
    long long* src = nullptr;
    double* srcv = nullptr;
    long long* rec = nullptr;
    double* damp = nullptr;
    int n_src = 0, n_rec = 0, cur = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    dim3 grid, block;
    long long nparts = 0;
    double* part_steps = nullptr;  // [steps][nparts] block partials of a run
    long long part_steps_cap = 0;
};

namespace {
template <typename T>
int fd_alloc(T** p, size_t n, char* errbuf, int errlen) {
    *p = nullptr;
    cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
    if (e != cudaSuccess) return fail(SFW_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e), errbuf, errlen);
    return 0;
}

FdParams fd_params(sfw_fdtd* h) {
    FdParams p{};
    p.nx = h->nx;
    p.ny = h->ny;
    p.nz = h->nz;
    p.s0 = h->s[0];
    p.s1 = h->s[1];
    p.s2 = h->s[2];
    p.c = h->c;
    p.part = h->part;
    return p;
}
}  // namespace

extern "C" int sfw_fdtd_create(int nx, int ny, int nz, const double* scales, const double* c, sfw_fdtd** out,
                               char* errbuf, int errlen) {
    *out = nullptr;
    if (nx < 1 || ny < 1 || nz < 1) return fail(SFW_ECONFIG, "grid dimensions must be positive", errbuf, errlen);
    if ((long long)nx * ny * nz >= (1LL << 31))
        return fail(SFW_ECONFIG, "fine grids are limited to 2^31 nodes (32-bit stencil offsets)", errbuf, errlen);
    auto* h = new sfw_fdtd();
    h->nx = nx;
    h->ny = ny;
    h->nz = nz;
    h->n = (long long)nx * ny * nz;
    for (int d = 0; d < 3; ++d) h->s[d] = scales[d];
    h->block = dim3(32, 8, 1);
    h->grid = dim3((nz + 31) / 32, (ny + 7) / 8, (nx + FD_XC - 1) / FD_XC);
    h->nparts = (long long)h->grid.x * h->grid.y * h->grid.z;
    int rc = 0;
    if ((rc = fd_alloc(&h->c, h->n, errbuf, errlen)) || (rc = fd_alloc(&h->U[0], h->n, errbuf, errlen)) ||
        (rc = fd_alloc(&h->U[1], h->n, errbuf, errlen)) || (rc = fd_alloc(&h->W, h->n, errbuf, errlen)) ||
        (rc = fd_alloc(&h->part, std::max<long long>(h->nparts, 2 * 1184), errbuf, errlen)) ||
        (rc = fd_alloc(&h->acc, 4, errbuf, errlen))) {
        delete h;
        return rc;
    }
    cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    cudaEventCreate(&h->ev0);
    cudaEventCreate(&h->ev1);
    SFW_CUDA_TRY(sfw_h2d(h->c, c, h->n * 8));
    *out = h;
    return 0;
}

// y = A x  (x, y HOST, length n) -- the row arithmetic of the solver, exposed for tests
extern "C" int sfw_fdtd_apply(sfw_fdtd* h, const double* x, double* y, char* errbuf, int errlen) {
    SFW_CUDA_TRY(cudaMemcpyAsync(h->W, x, h->n * 8, cudaMemcpyHostToDevice, h->stream));
    FdParams p = fd_params(h);
    p.u = h->W;
    p.out = h->U[0];
    k_fdtd<2><<<h->grid, h->block, 0, h->stream>>>(p);
    SFW_CUDA_TRY(cudaMemcpyAsync(y, h->U[0], h->n * 8, cudaMemcpyDeviceToHost, h->stream));
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    for (long long i = 0; i < h->n; ++i) y[i] = -y[i];  // kernel mode 2 writes -A x
    return 0;
}

// Largest eigenvalue of -A by power iteration from the HOST start vector v0 (already normalised,
// reference.py:26-63): w = -A v, lam = v.w, v = w/|w|, stop when |lam - lam_prev| <= tol |lam|.
extern "C" int sfw_fdtd_power(sfw_fdtd* h, const double* v0, double tol, int max_iter, double* lam_out,
                              int* iters_out, char* errbuf, int errlen) {
    double* v = h->U[0];
    double* w = h->W;
    SFW_CUDA_TRY(cudaMemcpyAsync(v, v0, h->n * 8, cudaMemcpyHostToDevice, h->stream));
    FdParams p = fd_params(h);
    const int nb = 1184;
    double lam = 0.0, res[2];
    int it = 0;
    for (; it < max_iter; ++it) {
        p.u = v;
        p.out = w;
        k_fdtd<2><<<h->grid, h->block, 0, h->stream>>>(p);
        k_fd_dots<<<nb, 256, 0, h->stream>>>(v, w, h->n, h->part);
        k_fd_dots_final<<<1, 1024, 0, h->stream>>>(h->part, nb, h->acc);
        SFW_CUDA_TRY(cudaMemcpyAsync(res, h->acc, 16, cudaMemcpyDeviceToHost, h->stream));
        SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
        const double nw = std::sqrt(res[1]);
        if (nw == 0.0) {
            *lam_out = 0.0;
            *iters_out = it + 1;
            return 0;
        }
        const double lam_new = res[0];
        k_fd_scale<<<nb, 256, 0, h->stream>>>(w, nw, h->n, v);
        if (it > 0 && std::fabs(lam_new - lam) <= tol * std::fabs(lam_new)) {
            lam = lam_new;
            ++it;
            *lam_out = lam;
            *iters_out = it;
            SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
            return 0;
        }
        lam = lam_new;
    }
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    *lam_out = lam;
    *iters_out = -max_iter;  // not converged (the caller logs, as reference.py:62 does)
    return 0;
}

// Sources (node index, value of source_vec there) and receiver rows; damping (HOST n) or null.
extern "C" int sfw_fdtd_setup(sfw_fdtd* h, int n_src, const long long* src_idx, const double* src_val, int n_rec,
                              const long long* rec_idx, const double* damping, char* errbuf, int errlen) {
    cudaFree(h->src);
    cudaFree(h->srcv);
    cudaFree(h->rec);
    cudaFree(h->damp);
    h->src = nullptr;
    h->srcv = nullptr;
    h->rec = nullptr;
    h->damp = nullptr;
    for (int i = 0; i < n_src; ++i)
        if (src_idx[i] < 0 || src_idx[i] >= h->n) return fail(SFW_ECONFIG, "source node outside the grid", errbuf, errlen);
    for (int i = 0; i < n_rec; ++i)
        if (rec_idx[i] < 0 || rec_idx[i] >= h->n) return fail(SFW_ECONFIG, "receiver node outside the grid", errbuf, errlen);
    int rc = 0;
    if ((rc = fd_alloc(&h->src, n_src, errbuf, errlen)) || (rc = fd_alloc(&h->srcv, n_src, errbuf, errlen)) ||
        (rc = fd_alloc(&h->rec, n_rec, errbuf, errlen)))
        return rc;
    if (n_src) {
        SFW_CUDA_TRY(sfw_h2d(h->src, src_idx, n_src * 8));
        SFW_CUDA_TRY(sfw_h2d(h->srcv, src_val, n_src * 8));
    }
    if (n_rec) SFW_CUDA_TRY(sfw_h2d(h->rec, rec_idx, n_rec * 8));
    if (damping) {
        if ((rc = fd_alloc(&h->damp, h->n, errbuf, errlen))) return rc;
        SFW_CUDA_TRY(sfw_h2d(h->damp, damping, h->n * 8));
    }
    h->n_src = n_src;
    h->n_rec = n_rec;
    return 0;
}

// Second-order start (reference.py:123-124): level 0 = u0, level -1 = u0 - dt v0 + (0.5 dt dt) a(u0, 0).
// u0 / v0 HOST (v0 may be null); f0 = source_fn(0).
extern "C" int sfw_fdtd_init(sfw_fdtd* h, double dt, const double* u0, const double* v0, double f0, char* errbuf,
                             int errlen) {
    h->cur = 0;
    if (u0)
        SFW_CUDA_TRY(cudaMemcpyAsync(h->U[0], u0, h->n * 8, cudaMemcpyHostToDevice, h->stream));
    else  // from rest: no host zeros to upload
        SFW_CUDA_TRY(cudaMemsetAsync(h->U[0], 0, h->n * 8, h->stream));
    if (v0) SFW_CUDA_TRY(cudaMemcpyAsync(h->W, v0, h->n * 8, cudaMemcpyHostToDevice, h->stream));
    FdParams p = fd_params(h);
    p.u = h->U[0];
    p.out = h->U[1];
    p.vel = v0 ? h->W : nullptr;
    p.dt = dt;
    p.half = (0.5 * dt) * dt;
    p.n_src = h->n_src;
    p.src_idx = h->src;
    p.src_val = h->srcv;
    p.f = f0;
    k_fdtd<1><<<h->grid, h->block, 0, h->stream>>>(p);
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    return 0;
}

// n_steps leapfrog steps.  ftab: HOST [n_steps] source_fn((k-1) dt) for step k = 1..n_steps.
// norms_out: HOST [n_steps] |u_k|^2 (fixed-order); rows_out: HOST [n_steps / record_every][n_rec]
// (u at the receivers after every record_every-th step).  *kernel_ms: CUDA-event time.
extern "C" int sfw_fdtd_run(sfw_fdtd* h, double dt, int n_steps, const double* ftab, int record_every,
                            double* norms_out, double* rows_out, float* kernel_ms, char* errbuf, int errlen) {
    if (n_steps <= 0) return 0;
    if (record_every < 1) return fail(SFW_ECONFIG, "record_every must be >= 1", errbuf, errlen);
    const long long nrec = n_steps / record_every;
    int rc = 0;
    if (h->norms_cap < n_steps) {
        cudaFree(h->norms);
        if ((rc = fd_alloc(&h->norms, n_steps, errbuf, errlen))) return rc;
        h->norms_cap = n_steps;
    }
    if (h->rows_cap < std::max(1LL, nrec * h->n_rec)) {
        cudaFree(h->rows);
        if ((rc = fd_alloc(&h->rows, std::max(1LL, nrec * h->n_rec), errbuf, errlen))) return rc;
        h->rows_cap = std::max(1LL, nrec * h->n_rec);
    }
    FdParams p = fd_params(h);
    p.dt = dt;
    p.dt2 = dt * dt;
    p.damping = h->damp;
    p.n_src = h->n_src;
    p.src_idx = h->src;
    p.src_val = h->srcv;
    if (h->part_steps_cap < (long long)n_steps * h->nparts) {
        cudaFree(h->part_steps);
        h->part_steps = nullptr;
        if ((rc = fd_alloc(&h->part_steps, (size_t)n_steps * h->nparts, errbuf, errlen))) return rc;
        h->part_steps_cap = (long long)n_steps * h->nparts;
    }
    p.n_rec = h->n_rec;
    p.rec = h->rec;
    // one launch per step: receivers are written by the stepping kernel and the per-step norm
    // partials kept, so the norms are reduced once after the loop (no per-step finish kernel)
    SFW_CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
    for (int k = 1; k <= n_steps; ++k) {
        p.u = h->U[h->cur];
        p.out = h->U[h->cur ^ 1];  // holds level k-2, receives level k
        p.f = h->n_src ? ftab[k - 1] : 0.0;
        p.part = h->part_steps + (size_t)(k - 1) * h->nparts;
        const bool rec = (k % record_every) == 0 && h->n_rec > 0;
        p.rows = rec ? h->rows + (k / record_every - 1) * h->n_rec : nullptr;
        k_fdtd<0><<<h->grid, h->block, 0, h->stream>>>(p);
        h->cur ^= 1;
    }
    k_fd_norms<<<n_steps, 1024, 0, h->stream>>>(h->part_steps, h->nparts, h->norms);
    SFW_CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
    if (norms_out) SFW_CUDA_TRY(cudaMemcpyAsync(norms_out, h->norms, n_steps * 8, cudaMemcpyDeviceToHost, h->stream));
    if (rows_out && nrec * h->n_rec)
        SFW_CUDA_TRY(cudaMemcpyAsync(rows_out, h->rows, nrec * h->n_rec * 8, cudaMemcpyDeviceToHost, h->stream));
    SFW_CUDA_TRY(cudaStreamSynchronize(h->stream));
    SFW_CUDA_TRY(cudaGetLastError());
    if (kernel_ms) cudaEventElapsedTime(kernel_ms, h->ev0, h->ev1);
    return 0;
}

// current and previous level (HOST n each, either may be null)
extern "C" int sfw_fdtd_state(sfw_fdtd* h, double* u_curr, double* u_prev, char* errbuf, int errlen) {
    if (u_curr) SFW_CUDA_TRY(cudaMemcpy(u_curr, h->U[h->cur], h->n * 8, cudaMemcpyDeviceToHost));
    if (u_prev) SFW_CUDA_TRY(cudaMemcpy(u_prev, h->U[h->cur ^ 1], h->n * 8, cudaMemcpyDeviceToHost));
    return 0;
}

extern "C" int sfw_fdtd_destroy(sfw_fdtd* h) {
    if (!h) return 0;
    void* ptrs[] = {h->c, h->U[0], h->U[1], h->W, h->part, h->acc, h->norms, h->rows, h->src, h->srcv, h->rec, h->damp,
                    h->part_steps};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return 0;
}
