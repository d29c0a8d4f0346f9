// Latency of the one-warp 20x20 Cholesky variants of ocpqp_fast.cuh, alone on
// one SM (cycles per factorization), plus the fp64 op latencies it is built from.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2003_02547_b200/csrc \
//      -I../../include -o chol chol.cu
#include <cstdio>

#include "ocpqp_fast.cuh"

using namespace ocpqp::fastk;
constexpr int NN = 20;

template <int V>
__global__ void kchol(const double* G, double* out, long long* t, int reps) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    long long c0 = 0, c1 = 0;
    for (int r = -1; r < reps; ++r) {
        if (r == 0) c0 = clock64();
        double row[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) row[j] = (lane < NN && j <= lane) ? G[lane * NN + j] + 1e-12 * acc : 0.0;
        double rin = 0.0;
        bool ok;
        if constexpr (V == 0) ok = warp_chol<NN>(row, lane, rin);
        else ok = warp_chol_rolled<NN>(row, lane, rin);
        acc += ok ? row[NN / 2] + rin : 1.0;
    }
    c1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) t[V] = (c1 - c0) / reps;
}

__global__ void kops(double* out, long long* t, int reps) {
    double x = 1.0 + threadIdx.x * 1e-9, y = 0.999999, s = 2.0 + threadIdx.x;
    long long c0 = clock64();
    for (int i = 0; i < reps; ++i) x = fma(x, y, 1e-7);
    long long c1 = clock64();
    t[2] = (c1 - c0) / reps;
    c0 = clock64();
    for (int i = 0; i < reps; ++i) s = rsqrt(s) + 1.5;
    c1 = clock64();
    t[3] = (c1 - c0) / reps;
    c0 = clock64();
    for (int i = 0; i < reps; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31);
    c1 = clock64();
    t[4] = (c1 - c0) / reps;
    out[threadIdx.x] = x + s;
}

int main() {
    double h[NN * NN];
    for (int i = 0; i < NN; ++i)
        for (int j = 0; j < NN; ++j) h[i * NN + j] = (i == j ? NN + 1.0 : 0.0) + 1.0 / (1.0 + i + j);
    double *G, *out;
    long long* t;
    cudaMalloc(&G, sizeof(h));
    cudaMalloc(&out, 4096);
    cudaMalloc(&t, 64);
    cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
    kchol<0><<<1, 32>>>(G, out, t, 64);
    kchol<1><<<1, 32>>>(G, out, t, 64);
    kops<<<1, 32>>>(out, t, 1024);
    cudaDeviceSynchronize();
    long long r[5];
    cudaMemcpy(r, t, sizeof(r), cudaMemcpyDeviceToHost);
    printf("warp_chol<20> unrolled: %lld cycles\nwarp_chol_rolled<20>: %lld cycles\n", r[0], r[1]);
    printf("dfma dep: %lld  rsqrt(double)+add dep: %lld  shfl.f64 dep: %lld cycles\n", r[2], r[3], r[4]);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
