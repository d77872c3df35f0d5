// Micro-benchmark: DMMA (mma.sync.m8n8k4.f64) issue rate per SM-cycle against the number of
// independent accumulator chains per warp (C) and warps per CTA (one CTA per SM), operands in
// registers (no LDS), and the single-chain dependent latency.  Sizes the ILP the multi-shot
// stepping kernel needs per warp.
//   build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/dmma_chain_bench tools/dmma_chain_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int C>
__global__ void k_chain(double* out, int iters, long long* cyc) {
    const int lane = threadIdx.x & 31;
    double acc[C][2];
#pragma unroll
    for (int i = 0; i < C; ++i) acc[i][0] = acc[i][1] = 1e-3 * (lane + i);
    const double a = 1e-3 * lane, b = 0.5;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) dmma(acc[i], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1234.5) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
void run(double* out, long long* cyc, int warps) {
    const int iters = 4000;
    k_chain<C><<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double dmmas = (double)C * iters * warps;
    printf("{\"chains\": %d, \"warps\": %d, \"dmma_per_sm_cycle\": %.4f, \"cycles_per_dmma_per_warp\": %.2f}\n", C,
           warps, dmmas / mx, (double)mx / ((double)C * iters));
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 148 * 8);
    for (int warps : {1, 4, 8, 16, 32}) {
        run<1>(out, cyc, warps);
        run<2>(out, cyc, warps);
        run<4>(out, cyc, warps);
        run<8>(out, cyc, warps);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
