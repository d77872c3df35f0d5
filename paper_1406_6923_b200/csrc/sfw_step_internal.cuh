// Internal state of a stepper handle, shared by sfw_step.cu and sfw_shots.cu.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "sfw_common.cuh"

namespace sfw {

template <typename T>
inline int dalloc(T** p, size_t n, char* errbuf, int errlen) {
    *p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
    if (e != cudaSuccess)
        return fail(SFW_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e), errbuf, errlen);
    return 0;
}

template <typename T>
inline int upload(T** p, const std::vector<T>& v, char* errbuf, int errlen) {
    int rc = dalloc(p, v.size(), errbuf, errlen);
    if (rc) return rc;
    if (!v.empty()) SFW_CUDA_TRY(cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return 0;
}

}  // namespace sfw

struct sfw_stepper {
    int n_sub = 0, m = 0, W = 0, BS = 0, n_src = 0, n_probe = 0, n_iface = 0;
    int grid = 0, nw = 0, ns = 0, smem = 0, cur = 0;
    long long state_len = 0, n_blocks = 0;
    double dt = 0;
    std::vector<int> layers;
    std::vector<long long> soff, src_len, prb_len;
    cudaStream_t stream = nullptr;
    cudaStream_t dstream = nullptr;  // probe-row downloads overlapped with later step chunks
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
    // k_step_lw (layer-warp resident kernel): launch shape + tagged face mailbox
    const void* klw = nullptr;
    int lw_smem = 0, lw_threads = 0, lw_groups = 1;
    double* ucoef = nullptr;  // k_ustep: chain blocks in the 16-B-pair layout
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
    int n_shots = 0, shot_smem = 0, shot_smem2 = 0;
    double* mmass = nullptr;  // multi-shot: per-subdomain interface mass blocks
    double* tcoef = nullptr;          // [n_blocks][TB] fragment-ordered 8x8 lower tiles
    int TB = 0;
    double *UM[2] = {nullptr, nullptr};
    double *mflux = nullptr, *macc1 = nullptr, *mfb = nullptr, *mnorm = nullptr, *mrows = nullptr;
    double* shot_vec = nullptr;        // [n_shots][K_s]
    int *shot_sub = nullptr, *shot_ptr = nullptr, *shot_ids = nullptr;
    long long* shot_voff = nullptr;
    double* shot_ftab = nullptr;
    long long shot_ftab_cap = 0, mrows_cap = 0, mnorm_cap = 0;
    int mcur = 0;
    int shot_smem3 = 0;               // k_step_ms3 dynamic smem (0: not used)
    int ms3_ng = 2, ms3_ns = 4;       // k_step_ms3 launch shape (subdomain groups, chain stages)
    unsigned int* sflags = nullptr;   // k_step_ms3: [n_sub][4] F_0 publication tags
    unsigned int stag = 0;            // k_step_ms3: last tag used
};

