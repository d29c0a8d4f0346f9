// Latency of the one-warp 20x20 Cholesky variants of ocpqp_fast.cuh, alone on
// one SM (cycles per factorization), plus the fp64 op latencies it is built from.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2003_02547_b200/csrc \
//      -I../../include -o chol chol.cu
#include <cstdio>

#include "ocpqp_fast.cuh"

using namespace ocpqp::fastk;
constexpr int NN = 20;

// the shift-register variant of Kern::chol_big (ocpqp_fast.cuh), rows from smem
__device__ __forceinline__ bool chol_shift(const double* Gu, double* Ls, double* rinv) {
    const int lane = threadIdx.x & 31;
    double r[NN];
#pragma unroll
    for (int m = 0; m < NN; ++m) r[m] = (lane < NN && m <= lane) ? Gu[lane * NN + m] : 0.0;
    bool ok = true;
#pragma unroll 1
    for (int k = 0; k < NN; ++k) {
        const double piv = __shfl_sync(0xffffffffu, r[0], k);
        ok = ok && (piv > 0.0);
        const double inv = rsqrt(piv);
        const double lik = lane == k ? piv * inv : r[0] * inv;
        if (lane == k) rinv[k] = inv;
        if (lane >= k && lane < NN) Ls[lane * NN + k] = lik;
#pragma unroll
        for (int m = 1; m < NN; ++m) {
            const int src = k + m < 32 ? k + m : 31;
            r[m - 1] = fma(-lik, __shfl_sync(0xffffffffu, lik, src), r[m]);
        }
        r[NN - 1] = 0.0;
    }
    return ok;
}

__global__ void kshift(const double* G, double* out, long long* t, int reps) {
    __shared__ double Gs[NN * NN], Ls[NN * NN], rv[32];
    for (int i = threadIdx.x; i < NN * NN; i += 32) Gs[i] = G[i];
    __syncwarp();
    double acc = 0.0;
    long long c0 = 0;
    for (int r = -1; r < reps; ++r) {
        if (r == 0) c0 = clock64();
        acc += chol_shift(Gs, Ls, rv) ? Ls[(threadIdx.x % NN) * NN] : 1.0;
        __syncwarp();
    }
    const long long c1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) t[5] = (c1 - c0) / reps;
}

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
    kshift<<<1, 32>>>(G, out, t, 64);
    cudaDeviceSynchronize();
    long long r[6];
    cudaMemcpy(r, t, sizeof(r), cudaMemcpyDeviceToHost);
    printf("warp_chol<20> unrolled: %lld cycles\nwarp_chol_rolled<20>: %lld cycles\n", r[0], r[1]);
    printf("dfma dep: %lld  rsqrt(double)+add dep: %lld  shfl.f64 dep: %lld cycles\n", r[2], r[3], r[4]);
    printf("chol_big shift-register variant: %lld cycles\n", r[5]);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
