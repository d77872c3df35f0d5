// Micro-benchmark: do DMMA (mma.sync.m8n8k4.f64) and FP64 ALU instructions (DFMA) share one pipe?
// 8 warps per CTA (2 per SMSP).  mode 0: all warps DMMA; mode 1: all warps DFMA; mode 2: even warps
// DMMA, odd warps DFMA (one of each per SMSP).  Reports per-warp cycles for a fixed instruction count.
//   build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/fp64_share_bench tools/fp64_share_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__global__ void k_share(int mode, int iters, long long* cyc, double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool do_dmma = mode == 0 || (mode == 2 && (warp & 4) == 0);
    double acc[8][2];
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 1e-3 * (lane + i);
    const double a = 1e-3 * lane, b = 0.999;
    __syncthreads();
    const long long t0 = clock64();
    if (do_dmma) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(acc[i], a, b);
    } else {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                acc[i][0] = fma(acc[i][0], b, a);
                acc[i][1] = fma(acc[i][1], b, a);
            }
    }
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1234.5) out[0] = s;
    if (lane == 0) cyc[blockIdx.x * 8 + warp] = t1 - t0;
}

int main() {
    long long* cyc;
    double* out;
    cudaMalloc(&cyc, 148 * 8 * 8);
    cudaMalloc(&out, 8);
    const int iters = 4000;
    for (int mode = 0; mode < 3; ++mode) {
        k_share<<<148, 256>>>(mode, iters, cyc, out);
        cudaDeviceSynchronize();
        long long c[148 * 8];
        cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
        double dm = 0, df = 0;
        int nd = 0, nf = 0;
        for (int i = 0; i < 148 * 8; ++i) {
            const int w = i % 8;
            const bool d = mode == 0 || (mode == 2 && (w & 4) == 0);
            if (d) { dm += c[i]; ++nd; } else { df += c[i]; ++nf; }
        }
        printf("{\"mode\": %d, \"dmma_cycles_per_inst\": %.2f, \"dfma_cycles_per_warp_inst\": %.2f}\n", mode,
               nd ? dm / nd / (8.0 * iters) : 0.0, nf ? df / nf / (16.0 * iters) : 0.0);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
