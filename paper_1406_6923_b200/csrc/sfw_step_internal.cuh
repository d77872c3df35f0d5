// Internal state of a stepper handle, shared by sfw_step.cu and sfw_shots.cu.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sfw_common.cuh"

namespace sfw {

template <typename T>
inline int upload(T** p, const std::vector<T>& v, char* errbuf, int errlen) {
    int rc = dalloc(p, v.size(), errbuf, errlen);
    if (rc) return rc;
    if (!v.empty()) SFW_CUDA_TRY(sfw_h2d(*p, v.data(), v.size() * sizeof(T)));
    return 0;
}


constexpr long long kChunkSlotBytes = 8LL << 20;  // one slot of the pinned row-staging ring

// Record boundaries 0 = b_0 < b_1 < ... < b_n = nrec of a run whose probe rows download while
// later chunks compute (sfw_step_run, sfw_wform_run).  One chunk when the rows are small; else
// n-1 equal chunks over the first 97% of the records and a short last chunk, whose download is
// the only one not hidden behind compute.  SFW_NO_CHUNK / SFW_CHUNK_BYTES / SFW_NCHUNK: hooks.
inline std::vector<long long> chunk_plan(long long nrec, long long row_bytes, bool have_rows) {
    std::vector<long long> b{0};
    long long chunk_min = 8LL << 20;
    if (const char* e = std::getenv("SFW_CHUNK_BYTES")) chunk_min = std::atoll(e);
    if (!have_rows || std::getenv("SFW_NO_CHUNK") || row_bytes < chunk_min || nrec < 16) {
        b.push_back(nrec);
        return b;
    }
    // >= 8 chunks, and enough that every chunk fits one staging slot (kChunkSlotBytes)
    int n = (int)std::min<long long>(64, std::max<long long>(8, 2 + row_bytes / kChunkSlotBytes));
    if (const char* e = std::getenv("SFW_NCHUNK")) n = std::max(2, std::min(64, std::atoi(e)));
    const long long tail = std::max(1LL, nrec * 3 / 100), head = nrec - tail;
    for (int c = 1; c < n; ++c) {
        const long long v = head * c / (n - 1);
        if (v > b.back()) b.push_back(v);
    }
    if (nrec > b.back()) b.push_back(nrec);
    return b;
}


}  // namespace sfw

struct sfw_stepper {
    int n_sub = 0, m = 0, W = 0, BS = 0, n_src = 0, n_probe = 0, n_iface = 0;
    int grid = 0, nw = 0, ns = 0, smem = 0, cur = 0;
    long long state_len = 0, n_blocks = 0;
    double dt = 0;
    std::vector<int> layers;
    std::vector<int> src_subs_h;  // subdomains that carry a source (host copy, ascending)
    int* src_subs = nullptr;      // same, on the device
    std::vector<long long> soff, src_len, prb_len;
    cudaStream_t stream = nullptr;
    cudaStream_t dstream = nullptr;  // probe-row downloads overlapped with later step chunks
    double* pin = nullptr;            // 2-slot pinned staging ring for those downloads
    size_t pin_cap = 0;               // bytes
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double* coef = nullptr;
    long long* seq = nullptr;
    int *seq_ptr = nullptr, *wsub = nullptr, *wsub_ptr = nullptr, *cta_sub_ptr = nullptr;
    int *d_layers = nullptr, *nbr = nullptr, *mass_idx = nullptr, *ncta_ptr = nullptr, *ncta = nullptr;
    long long* d_soff = nullptr;
    double* mass = nullptr;
    double *U[2] = {nullptr, nullptr}, *S[2] = {nullptr, nullptr}, *V0 = nullptr, *acc1 = nullptr, *fbuf = nullptr;
    int *src_ptr = nullptr, *src_ids = nullptr;
    double* src_vec = nullptr;
    long long* src_voff = nullptr;
    double* ftab = nullptr;
    long long ftab_cap = 0;
    int *prb_ptr = nullptr, *prb_ids = nullptr, *prb_tap = nullptr;
    double* prb_w = nullptr;
    long long* prb_woff = nullptr;
    double* rows = nullptr;
    long long rows_cap = 0;
    double *sub_norm = nullptr, *norm_part = nullptr, *norms = nullptr;
    long long norms_cap = 0;  // capacity of norms (grown, never freed per run: cudaFree would sync the device)
    long long norm_cap = 0;
    unsigned int* bar = nullptr;
    double* scales = nullptr;  // dense G_j (energy), may be null
    double* gam_dense = nullptr;  // dense Gamma_j (energy)
    bool evict_first = true;
    bool uniform = false;
    int L = 0;
    const void* kfn = nullptr;
    const void* kres = nullptr;
    int res_smem = 0, res_nw = 0, res_pmax = 0, res_pdense = 0;
    // warp-per-subdomain kernels (k_step_sw, k_ustep): launch shape + tagged face mailbox
    const void* klw = nullptr;
    int lw_smem = 0, lw_threads = 0, lw_groups = 1;
    double* ucoef = nullptr;  // k_ustep: chain blocks in the 16-B-pair layout
    double* swimg = nullptr;  // k_step_sw: every subdomain's 2L blocks pre-expanded to the SMEM image
    int BS2 = 0;
    bool ustep = false;
    int n_interior = 0;  // subdomains with all six faces shared
    unsigned long long* mbox = nullptr;
    unsigned int tag_base = 0;
    int max_src_sub = 0;  // most sources injected into one subdomain
    std::vector<int> cta_ptr_h;
    unsigned long long* tprof = nullptr;
    size_t tprof_n = 0;
    double* flux = nullptr;
    double* sq = nullptr;
    // multi-shot mode (sfw_shots_*): S independent wavefields, DMMA tile-packed chain blocks
    int n_shots = 0, shot_smem2 = 0;
    std::vector<int> nbr_h;           // host copy of the face-neighbour table [n_sub][6]
    int mt_grid = 0, mt_nst = 0, mt_team_smem = 0;  // k_step_mt: teams (two per CTA), ring stages, bytes per team
    int *mt_cta_ptr = nullptr, *mt_ncta_ptr = nullptr, *mt_ncta = nullptr;
    int mt_nsmax = 0;
    unsigned int* mt_flags = nullptr;
    double* mmass = nullptr;  // multi-shot: per-subdomain interface mass tiles
    double* tcoef = nullptr;          // [n_blocks][TB] swizzled 8x8 lower tiles
    int TB = 0;
    double *UM[2] = {nullptr, nullptr};
    double *mflux = nullptr, *macc1 = nullptr, *mfb = nullptr, *mnorm = nullptr, *mrows = nullptr;
    double* shot_vec = nullptr;        // [n_shots][K_s]
    int *shot_sub = nullptr, *shot_ptr = nullptr, *shot_ids = nullptr;
    long long* shot_voff = nullptr;
    double* shot_ftab = nullptr;
    long long shot_ftab_cap = 0, mrows_cap = 0, mnorm_cap = 0;
    int mcur = 0;
};

namespace sfw {
// Pinned staging for download_rows_overlapped, grown before any launch of the run (a pinned
// allocation must not wait behind the run it is meant to overlap).
inline cudaError_t ensure_row_staging(sfw_stepper* h, const std::vector<long long>& plan, long long n_probe) {
    size_t maxb = 0;
    for (size_t c = 0; c + 1 < plan.size(); ++c) maxb = std::max<size_t>(maxb, (size_t)(plan[c + 1] - plan[c]) * n_probe * 8);
    if (h->pin_cap >= 2 * maxb && h->pin) return cudaSuccess;
    if (h->pin) cudaFreeHost(h->pin);
    h->pin = nullptr;
    h->pin_cap = 0;
    cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&h->pin), 2 * maxb);
    if (e == cudaSuccess) h->pin_cap = 2 * maxb;
    return e;
}

// Rows [plan[c], plan[c+1]) of chunk c (n_probe doubles per record) go device -> pinned slot c&1
// on dstream once chunk c's event fires, then pinned -> the caller's pageable array on the host
// while the DMA of chunk c+1 and the compute of later chunks proceed.
inline cudaError_t download_rows_overlapped(sfw_stepper* h, const std::vector<long long>& plan,
                                            const std::vector<cudaEvent_t>& evs, const double* dev, double* host,
                                            long long n_probe) {
    const int n = (int)plan.size() - 1;
    const size_t slot = h->pin_cap / 2 / 8;
    std::vector<cudaEvent_t> done(n, nullptr);
    cudaError_t err = cudaSuccess;
    auto issue = [&](int c) {
        const size_t bytes = (size_t)(plan[c + 1] - plan[c]) * n_probe * 8;
        cudaEventCreateWithFlags(&done[c], cudaEventDisableTiming);
        cudaStreamWaitEvent(h->dstream, evs[c], 0);
        if (bytes) {
            cudaError_t e = cudaMemcpyAsync(h->pin + (c & 1) * slot, dev + plan[c] * n_probe, bytes,
                                            cudaMemcpyDeviceToHost, h->dstream);
            if (e != cudaSuccess) err = e;
        }
        cudaEventRecord(done[c], h->dstream);
    };
    issue(0);
    for (int c = 1; c <= n; ++c) {
        if (c < n) issue(c);
        const int p = c - 1;
        cudaError_t e = cudaEventSynchronize(done[p]);
        if (e != cudaSuccess) err = e;
        const size_t bytes = (size_t)(plan[p + 1] - plan[p]) * n_probe * 8;
        if (bytes && err == cudaSuccess) std::memcpy(host + plan[p] * n_probe, h->pin + (p & 1) * slot, bytes);
    }
    for (cudaEvent_t e : done) cudaEventDestroy(e);
    return err;
}

}  // namespace sfw


