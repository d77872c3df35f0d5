// Shared helpers for the sm_100a kernels of libsfw_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <cstdlib>
#include <string>

#include "../../include/sfw_b200.h"

namespace sfw {

// ---- error plumbing -------------------------------------------------------

void set_error(int code, const std::string& msg);
int fail(int code, const std::string& msg, char* errbuf, int errlen);

// Pageable host -> device copy that has landed when it returns.  cudaMemcpy from pageable memory
// may return with the DMA still in flight on the legacy stream, and kernels on the library's
// non-blocking streams do not order with that stream.
inline cudaError_t sfw_h2d(void* dst, const void* src, size_t bytes) {
    cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(0);
}

#define SFW_CUDA_TRY(expr)                                                            \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess)                                                        \
            return ::sfw::fail(SFW_ECUDA, std::string(#expr ": ") + cudaGetErrorString(_e), \
                               errbuf, errlen);                                       \
    } while (0)

// ---- device allocation (every library buffer; SFW_POISON debug fill) ---------

inline int g_wform_scope = 0;  // debug poisoning: > 0 while a W-form entry point allocates

template <typename T>
inline int dalloc(T** p, size_t n, char* errbuf, int errlen) {
    *p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
    if (e != cudaSuccess)
        return fail(SFW_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e), errbuf, errlen);
    if (const char* pz = std::getenv("SFW_POISON")) {  // debug: fresh buffers read as NaN until written
        const bool w = g_wform_scope > 0;
        if (pz[0] == 'a' || (pz[0] == 'w' && w) || (pz[0] == 's' && !w)) {
            // legacy-stream memset + a legacy-stream sync only: library kernels run on non-blocking
            // streams and are not drained here (every H2D copy already syncs the legacy stream)
            cudaMemset(*p, 0xFF, n * sizeof(T));
            cudaStreamSynchronize(cudaStreamLegacy);
        }
    }
    return 0;
}

// ---- PTX wrappers: mbarrier + 1-D bulk async copy (TMA engine) -------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// non-blocking probe (try_wait may suspend the thread for a while)
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// try_wait with a suspend-time hint (ns): the thread sleeps in hardware until the phase completes
// (or the hint elapses), so a producer lane waiting on a full ring takes no issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!ok);
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ---- grid-wide split barrier (monotone counter, release/acquire at gpu scope) --

__device__ __forceinline__ void grid_arrive(unsigned int* ctr) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_wait(const unsigned int* ctr, unsigned int target) {
    while (ld_acquire(ctr) < target) {
        __nanosleep(32);
    }
    __threadfence();
}

// neighbour-only step flags: CTA c publishes "phase A of step k done" as flags[c] = k
// (release, gpu scope); a CTA waits only for the CTAs that own its subdomains'
// face neighbours (acquire).  Double-buffered face data make this sufficient.
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Called by one thread after a __syncthreads(): bar.sync orders the CTA's prior
// writes before this thread's release store (cumulativity), so no extra fence.
__device__ __forceinline__ void flag_publish(unsigned int* flags, unsigned int k) {
    st_release(flags + blockIdx.x, k);
}

// called by one full warp
__device__ __forceinline__ void flags_wait(const unsigned int* flags, const int* list, int n, unsigned int k,
                                           int lane) {
    for (int i = lane; i < n; i += 32) {
        const unsigned int* f = flags + list[i];
        while (ld_acquire(f) < k) {
        }
    }
    __syncwarp();  // acquire loads above; the caller's __syncthreads() publishes them to the CTA
}

// fixed-order warp sum (butterfly; identical order on every call -> deterministic)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace sfw
