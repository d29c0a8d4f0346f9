// Latency micro-benchmarks for the fp64 building blocks of the team kernel
// (single warp / single CTA, clock64 deltas).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 256
__global__ void k(double* out, long long* t, double x0, int tm) {
    __shared__ double sm[1024];
    __shared__ double buf[64];
    const int tid = threadIdx.x;
    for (int i = tid; i < 1024; i += blockDim.x) sm[i] = 1.0 + 1e-3 * i;
    __syncthreads();
    double x = x0 + tid * 1e-9, y = 1.0000001;
    long long c0, c1;
    // 1 DFMA chain
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) { x = fma(x, y, 1e-7); x = fma(x, y, 1e-7); x = fma(x, y, 1e-7); x = fma(x, y, 1e-7); }
    c1 = clock64(); if (tid == 0) t[0] = (c1 - c0);
    // 2 LDS dependent chain (address from loaded value)
    int idx = tid & 7;
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) { double v = sm[idx]; idx = ((int)v) & 7; v = sm[idx + 8]; idx = ((int)v) & 7; }
    c1 = clock64(); if (tid == 0) t[1] = (c1 - c0); x += idx;
    // 3 shfl chain
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) { x = __shfl_xor_sync(0xffffffff, x, 1); x = __shfl_xor_sync(0xffffffff, x, 2); }
    c1 = clock64(); if (tid == 0) t[2] = (c1 - c0);
    // 4 sqrt chain
    double s = 2.0 + tid;
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) { s = sqrt(s) + 1.5; s = sqrt(s) + 1.5; }
    c1 = clock64(); if (tid == 0) t[3] = (c1 - c0); x += s;
    // 5 rsqrt chain
    s = 2.0 + tid;
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) { s = rsqrt(s) + 1.5; s = rsqrt(s) + 1.5; }
    c1 = clock64(); if (tid == 0) t[4] = (c1 - c0); x += s;
    // 6 div chain
    s = 2.0 + tid;
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) { s = 3.0 / s + 1.5; s = 3.0 / s + 1.5; }
    c1 = clock64(); if (tid == 0) t[5] = (c1 - c0); x += s;
    // 7 syncthreads round trip (STS + bar + LDS)
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) {
        buf[tid & 63] = x; __syncthreads(); x = buf[(tid + 1) & 63] * 0.5 + 1e-3; __syncthreads();
    }
    c1 = clock64(); if (tid == 0) t[6] = (c1 - c0);
    // 8 syncwarp round trip (STS + syncwarp + LDS)
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) {
        buf[tid & 63] = x; __syncwarp(); x = buf[(tid ^ 1) & 63] * 0.5 + 1e-3; __syncwarp();
    }
    c1 = clock64(); if (tid == 0) t[7] = (c1 - c0);
    // 9 global (L1-hit) dependent load chain
    const double* g = out + 64;
    int gi = tid & 7;
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) { double v = g[gi]; gi = ((int)v) & 7; v = g[gi + 8]; gi = ((int)v) & 7; }
    c1 = clock64(); if (tid == 0) t[8] = (c1 - c0); x += gi;
    // 10 volatile global chain (L2)
    volatile double* vg = out + 64;
    gi = tid & 7;
    c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N_IT; ++i) { double v = vg[gi * 16]; gi = ((int)v) & 7; v = vg[gi * 16 + 8]; gi = ((int)v) & 7; }
    c1 = clock64(); if (tid == 0) t[9] = (c1 - c0); x += gi;
    out[tid] = x;
}
int main() {
    double* d; long long* t; cudaMalloc(&d, 1 << 20); cudaMalloc(&t, 128);
    cudaMemset(d, 0, 1 << 20);
    const char* nm[] = {"dfma", "lds(dep)", "shfl", "sqrt+add", "rsqrt+add", "div+add", "sts+bar+lds+bar (64thr)",
                        "sts+syncwarp+lds+syncwarp", "ldg L1 (dep)", "ld.volatile (dep)"};
    const double per[] = {4, 2, 2, 2, 2, 2, 1, 1, 2, 2};
    for (int th : {32, 64}) {
        k<<<1, th>>>(d, t, 1.0, 0); cudaDeviceSynchronize();
        k<<<1, th>>>(d, t, 1.0, 0);
        long long h[10]; cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
        printf("threads=%d\n", th);
        for (int i = 0; i < 10; ++i) printf("  %-30s %7.1f cyc/op\n", nm[i], h[i] / (N_IT * per[i]));
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
