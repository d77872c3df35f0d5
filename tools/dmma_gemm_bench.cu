// Micro-benchmark: the multi-shot kernels' inner GEMM (Y(56 x 8) = B(56 x 56, symmetric, lower 8x8
// tiles in DMMA fragment order) X(56 x 8)), operands from shared memory exactly as k_step_ms4 reads
// them: per k-step one LDS of X and 7 LDS of chain-block fragments feeding 7 DMMA chains.  Reports
// DMMA per SM-cycle against warps per CTA (1 CTA per SM), to tell the GEMM loop's own ceiling from
// the stepping kernel's other costs.
//   build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/dmma_gemm_bench tools/dmma_gemm_bench.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

constexpr int RT = 7, LDX = 12;

template <int XSTORE>
__global__ void k_gemm(double* out, int iters, long long* cyc) {
    extern __shared__ double sm[];
    double* tiles = sm;                         // 28 x 64
    double* X = sm + 28 * 64;                   // per warp 56 x LDX
    for (int i = threadIdx.x; i < 28 * 64 + (blockDim.x / 32) * 56 * LDX; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* Xs = X + warp * 56 * LDX;
    const int r0 = lane >> 2;
    int tr[2];
    for (int h = 0; h < 2; ++h) {
        const int r = 4 * h + (lane & 3), c = lane >> 2;
        tr[h] = (c >> 2) * 32 + r * 4 + (c & 3);
    }
    double keep[RT][2];
    for (int i = 0; i < RT; ++i) keep[i][0] = keep[i][1] = 0.0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        double acc[RT][2];
#pragma unroll
        for (int i = 0; i < RT; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
        for (int kap = 0; kap < 2 * RT; ++kap) {
            const int Kt = kap >> 1, h = kap & 1;
            const double b = Xs[(4 * kap + (lane & 3)) * LDX + r0];
#pragma unroll
            for (int I = 0; I < RT; ++I) {
                const double a = (I >= Kt) ? tiles[(I * (I + 1) / 2 + Kt) * 64 + h * 32 + lane]
                                           : tiles[(Kt * (Kt + 1) / 2 + I) * 64 + tr[h]];
                dmma(acc[I], a, b);
            }
        }
        if (XSTORE) {  // write the result back as the next X (as the stepping kernel does)
            __syncwarp();
#pragma unroll
            for (int i = 0; i < RT; ++i)
                *reinterpret_cast<double2*>(Xs + (8 * i + r0) * LDX + 2 * (lane & 3)) =
                    make_double2(acc[i][0] * 1e-3, acc[i][1] * 1e-3);
            __syncwarp();
        } else {
#pragma unroll
            for (int i = 0; i < RT; ++i) {
                keep[i][0] += acc[i][0];
                keep[i][1] += acc[i][1];
            }
        }
    }
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < RT; ++i) s += keep[i][0] + keep[i][1];
    if (s == 1234.5) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int XS>
void run(double* out, long long* cyc, int warps) {
    const int iters = 2000;
    const size_t smem = (28 * 64 + warps * 56 * LDX) * 8;
    cudaFuncSetAttribute(k_gemm<XS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_gemm<XS><<<148, warps * 32, smem>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("{\"xstore\": %d, \"warps\": %d, \"dmma_per_sm_cycle\": %.4f}\n", XS, warps, 98.0 * iters * warps / mx);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 148 * 8);
    for (int w : {4, 8, 12, 16}) {
        run<0>(out, cyc, w);
        run<1>(out, cyc, w);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
