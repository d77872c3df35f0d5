// Negative control of the config-4 repeatability investigation (config 4; the cause was a missing
// proxy fence before the ring refills, not this): does a queued
// mma.sync.m8n8k4.f64 read its operand registers after later instructions of the same warp have
// overwritten them?  Every warp of every CTA computes the SAME sequence of GEMM-like products from the
// same shared-memory operands (7 independent accumulator chains, B fragments loaded one k-step ahead into
// a two-deep register buffer, no holds), so every warp must produce the same bits as a run with one
// warp per SMSP.  Reports, per warps-per-CTA, how many warp results differ from that reference over
// repeated launches.
//   build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/dmma_hazard_bench tools/dmma_hazard_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

constexpr int RT = 7, KS = 13, NB = KS * RT;  // k-steps and B fragments of one product

__global__ void k_hazard(double* out, int rounds) {
    extern __shared__ double sm[];
    double* B = sm;             // [NB][32] fragment-ordered
    double* A = sm + NB * 32;   // [KS][32]
    for (int i = threadIdx.x; i < (NB + KS) * 32; i += blockDim.x)
        sm[i] = 1.0 + 1e-3 * ((i * 2654435761u) % 1013) - 0.5;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double x[KS];
#pragma unroll
    for (int k = 0; k < KS; ++k) x[k] = A[k * 32 + lane];
    double acc[RT][2];
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
        for (int t = 0; t < RT; ++t) acc[t][0] = acc[t][1] = 0.0;
        double bb[2][RT];
#pragma unroll
        for (int t = 0; t < RT; ++t) bb[0][t] = B[t * 32 + lane];
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            if (k + 1 < KS) {
#pragma unroll
                for (int t = 0; t < RT; ++t) bb[(k + 1) & 1][t] = B[((k + 1) * RT + t) * 32 + lane];
            }
#pragma unroll
            for (int t = 0; t < RT; ++t) dmma(acc[t], x[k], bb[k & 1][t]);
        }
        // the next product's A operands from this one's results (as the layer sweep does), kept O(1)
#pragma unroll
        for (int k = 0; k < KS; ++k) x[k] = 0.5 * x[k] + 1e-3 * acc[k % RT][k & 1];
    }
    double* o = out + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32 * (KS + 2 * RT) + lane;
#pragma unroll
    for (int k = 0; k < KS; ++k) o[k * 32] = x[k];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
        o[(KS + 2 * t) * 32] = acc[t][0];
        o[(KS + 2 * t + 1) * 32] = acc[t][1];
    }
}

int main(int argc, char** argv) {
    const int rounds = argc > 1 ? atoi(argv[1]) : 2000, reps = argc > 2 ? atoi(argv[2]) : 50;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t per_warp = 32 * (KS + 2 * RT), smem = (NB + KS) * 32 * 8;
    cudaFuncSetAttribute(k_hazard, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    std::vector<double> ref(per_warp), got;
    double* d = nullptr;
    cudaMalloc(&d, (size_t)nsm * 32 * per_warp * 8);
    // reference: one warp per SMSP, one CTA
    k_hazard<<<1, 128, smem>>>(d, rounds);
    cudaMemcpy(ref.data(), d, per_warp * 8, cudaMemcpyDeviceToHost);
    for (int wpc : {4, 8, 12, 16, 24, 32}) {
        long long bad = 0, total = 0;
        for (int rep = 0; rep < reps; ++rep) {
            k_hazard<<<nsm, wpc * 32, smem>>>(d, rounds);
            got.resize((size_t)nsm * wpc * per_warp);
            cudaMemcpy(got.data(), d, got.size() * 8, cudaMemcpyDeviceToHost);
            for (int w = 0; w < nsm * wpc; ++w) {
                ++total;
                if (memcmp(&got[(size_t)w * per_warp], ref.data(), per_warp * 8) != 0) ++bad;
            }
        }
        printf("warps per CTA %2d (per SMSP %d): %lld of %lld warp results differ from the 1-warp-per-SMSP reference\n", wpc,
               wpc / 4, bad, total);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("cuda: %s\n", cudaGetErrorString(e));
    return 0;
}
