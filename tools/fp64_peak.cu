// FP64 peak micro-benchmark for the roofline denominators (MEASURED_PEAKS.json has no fp64 entry).
//
//   build: make tools   ->  build/fp64_peak
//   run  : build/fp64_peak   (one JSON line: DMMA m8n8k4 and DFMA TFLOP/s, burst, CUDA events)
//
// DMMA: every warp keeps 8 independent m8n8k4 accumulators (2 doubles per lane each) and
// issues mma.sync.aligned.m8n8k4.row.col.f64 back to back: 2*8*8*4 = 512 flops per MMA.
// DFMA: 16 independent fma chains per thread, 2 flops per fma.
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k_dmma(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = fma(c[i], b, a);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int sms = pr.multiProcessorCount;
    double best_mma = 0, best_fma = 0;
    int best_mma_w = 0, best_fma_w = 0;
    for (int cfg = 0; cfg < 8; ++cfg) {
        const int warps = (cfg & 3) == 0 ? 4 : (cfg & 3) == 1 ? 8 : (cfg & 3) == 2 ? 16 : 32;
        const int iters = 20000;
        const int blocks = sms * (cfg < 4 ? 1 : 2);
        k_dmma<<<blocks, warps * 32>>>(out, 100);
        cudaEventRecord(e0);
        k_dmma<<<blocks, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 512.0 * 8 * iters * (double)blocks * warps;
        const double tf = fl / (ms * 1e-3) / 1e12;
        if (tf > best_mma) best_mma = tf, best_mma_w = warps * (cfg < 4 ? 1 : 2);
        k_dfma<<<blocks, warps * 32>>>(out, 100);
        cudaEventRecord(e0);
        k_dfma<<<blocks, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl2 = 2.0 * 16 * iters * (double)blocks * warps * 32;
        const double tf2 = fl2 / (ms * 1e-3) / 1e12;
        if (tf2 > best_fma) best_fma = tf2, best_fma_w = warps * (cfg < 4 ? 1 : 2);
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"dmma_f64_tflops\": %.3f, \"dmma_warps_per_sm\": %d, "
           "\"dfma_f64_tflops\": %.3f, \"dfma_warps_per_sm\": %d, \"how\": \"mma.sync m8n8k4 f64 (8 indep. "
           "accumulators/warp) and fma.f64 (16 chains/thread), 1 or 2 CTAs/SM x 4-32 warps, best, CUDA events, "
           "burst\", \"cuda\": \"%s\"}\n",
           pr.name, sms, best_mma, best_mma_w, best_fma, best_fma_w, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
