// DMMA (mma.sync m8n8k4 f64) latency / throughput micro-benchmark on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma dmma.cu && ./dmma
// Prints cycles per DMMA for a dependent chain (1 accumulator) and for
// ACC independent accumulators per warp, at several warps per CTA.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int ACC>
__global__ void k(double* out, long long* t, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    double d[ACC][2];
#pragma unroll
    for (int i = 0; i < ACC; ++i) d[i][0] = d[i][1] = i * 1e-3;
    __syncthreads();
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i) dmma(d[i][0], d[i][1], a, b);
    }
    const long long c1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += d[i][0] + d[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) t[blockIdx.x] = c1 - c0;
}

template <int ACC>
void run(int warps, double* out, long long* t) {
    const int iters = 4096;
    k<ACC><<<1, 32 * warps>>>(out, t, iters);
    k<ACC><<<1, 32 * warps>>>(out, t, iters);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, t, sizeof(h), cudaMemcpyDeviceToHost);
    const double per_warp = (double)h / (iters * ACC);
    printf("acc %2d warps %2d: %7.2f cycles per DMMA per warp, SM rate %6.2f FMA/clk\n", ACC, warps,
           per_warp, 256.0 * warps / per_warp);
}

int main() {
    double* out;
    long long* t;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&t, 1 << 12);
    for (int w : {1, 2, 4, 8, 16}) {
        run<1>(w, out, t);
        run<2>(w, out, t);
        run<4>(w, out, t);
        run<8>(w, out, t);
    }
    return 0;
}
