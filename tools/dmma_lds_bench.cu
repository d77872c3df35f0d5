// Micro-benchmark: DMMA throughput of LDS-fed m8n8k4 products, as the multi-shot stepping
// kernels issue them (per k-step: 2 quad shuffles build the A fragment, then one LDS.64 of a
// chain-block fragment per row tile and one DMMA).  Reports DMMA per SM-cycle against the
// number of warps per CTA (one CTA per SM), to size the warp count of k_step_ms*.
//   build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/dmma_lds_bench tools/dmma_lds_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int RT, bool SHFL>
__global__ void k_bench(double* out, int iters, long long* cyc) {
    extern __shared__ double tiles[];  // 28 tiles x 64 doubles
    for (int i = threadIdx.x; i < 28 * 64; i += blockDim.x) tiles[i] = 1e-3 * (i % 97);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double P[RT][2], C[RT][2];
#pragma unroll
    for (int I = 0; I < RT; ++I) P[I][0] = P[I][1] = 1e-3 * (lane + I);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int I = 0; I < RT; ++I) C[I][0] = C[I][1] = 0.0;
#pragma unroll
        for (int kap = 0; kap < 2 * RT; ++kap) {
            const int Ip = kap >> 1, h = kap & 1;
            double xa = P[Ip][h];
            if (SHFL) {
                const double v0 = __shfl_sync(0xffffffffu, P[Ip][0], (lane & ~3) | (2 * h + ((lane & 3) >> 1)));
                const double v1 = __shfl_sync(0xffffffffu, P[Ip][1], (lane & ~3) | (2 * h + ((lane & 3) >> 1)));
                xa = (lane & 1) ? v1 : v0;
            }
#pragma unroll
            for (int I = 0; I < RT; ++I) {
                const int Kt = Ip;
                const double b = (I >= Kt) ? tiles[(I * (I + 1) / 2 + Kt) * 64 + h * 32 + lane]
                                           : tiles[(Kt * (Kt + 1) / 2 + I) * 64 + ((lane >> 2) >> 2) * 32 + (4 * h + (lane & 3)) * 4 + ((lane >> 2) & 3)];
                dmma(C[I], xa, b);
            }
        }
#pragma unroll
        for (int I = 0; I < RT; ++I) {
            P[I][0] = C[I][0] * 1e-9 + P[I][0];
            P[I][1] = C[I][1] * 1e-9 + P[I][1];
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int I = 0; I < RT; ++I) s += P[I][0] + P[I][1];
    if (s == 1234.5) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(k_bench<7, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 28 * 64 * 8);
    cudaFuncSetAttribute(k_bench<7, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 28 * 64 * 8);
    const int iters = 2000;
    for (int shfl = 0; shfl < 2; ++shfl)
        for (int warps : {2, 4, 8, 12, 16, 24, 32}) {
            if (shfl)
                k_bench<7, true><<<148, warps * 32, 28 * 64 * 8>>>(out, iters, cyc);
            else
                k_bench<7, false><<<148, warps * 32, 28 * 64 * 8>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            long long c[148];
            cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
            const double dmmas = 98.0 * iters * warps;
            printf("{\"shfl\": %d, \"warps\": %d, \"dmma_per_sm_cycle\": %.3f}\n", shfl, warps, dmmas / mx);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
