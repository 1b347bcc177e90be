// Single-warp latency probe for K4's dependent chains (sm_100a): cycles per
// dependent DFMA, per dependent DADD, per 64-bit __shfl_sync broadcast and
// per shuffle + DFMA step (the FGS coordinate chain).  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat_probe tools/lat_probe.cu && /tmp/lat_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void probe(double *out, long long *cyc, double a, double b)
{
    double x = a + threadIdx.x * 1e-3;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    double y = x;
#pragma unroll 64
    for (int i = 0; i < N; ++i) y = y + b;
    long long t2 = clock64();
    double z = y;
#pragma unroll 64
    for (int i = 0; i < N; ++i) z = __shfl_sync(0xffffffffu, z, (i + 1) & 31);
    long long t3 = clock64();
    double w = z;
#pragma unroll 64
    for (int i = 0; i < N; ++i) w = fma(-a, __shfl_sync(0xffffffffu, w, i & 31), w);
    long long t4 = clock64();
    out[threadIdx.x] = w;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
        cyc[3] = t4 - t3;
    }
}

int main()
{
    double *out;
    long long *cyc, h[4];
    cudaMalloc(&out, 32 * sizeof(double));
    cudaMalloc(&cyc, 4 * sizeof(long long));
    for (int rep = 0; rep < 3; ++rep) probe<<<1, 32>>>(out, cyc, 0.999999, 1e-9);
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op (one warp, %d-long chains):\n", N);
    printf("  DFMA              %.2f\n", (double)h[0] / N);
    printf("  DADD              %.2f\n", (double)h[1] / N);
    printf("  SHFL (64-bit)     %.2f\n", (double)h[2] / N);
    printf("  SHFL + DFMA step  %.2f\n", (double)h[3] / N);
    return cudaGetLastError() != cudaSuccess;
}
