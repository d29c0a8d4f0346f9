// FP64 peak microbenchmarks (roofline denominators; MEASURED_PEAKS.json has
// no fp64 entry).  Exported through the C ABI as ocpqp_fp64_peak().
//   * DFMA: 8 independent FMA chains per thread, 148 x k CTAs of 256 threads;
//   * DMMA: mma.sync.m8n8k4.f64 (the only fp64 tensor-core path on sm_100a,
//     lowered by ptxas to DMMA.8x8x4), 4 independent accumulators per warp.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double seed) {
    double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_dmma(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
    double d[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) { d[j][0] = 0.0; d[j][1] = 0.0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            asm volatile(
                "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                : "+d"(d[j][0]), "+d"(d[j][1])
                : "d"(a), "d"(b));
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1];
    if (s == 12345.678) out[blockIdx.x] = s;
}

}  // namespace

extern "C" int ocpqp_fp64_peak(double* dfma_tflops, double* dmma_tflops) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -4;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double) * 4096) != cudaSuccess) return -4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 8, threads = 256;
    // DFMA: flops = grid * threads * iters * 8 chains * 8 unroll * 2
    int iters = 4096;
    k_dfma<<<grid, threads>>>(out, 64, 1.0);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<grid, threads>>>(out, iters, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    if (dfma_tflops)
        *dfma_tflops = (double)grid * threads * iters * 128.0 / (best * 1e-3) / 1e12;
    // DMMA: flops per mma = 2 * 8 * 8 * 4 = 512 per warp-instruction
    iters = 2048;
    k_dmma<<<grid, threads>>>(out, 16);
    best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dmma<<<grid, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    if (dmma_tflops)
        *dmma_tflops = (double)grid * (threads / 32) * iters * 4 * 512.0 / (best * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}
