#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma(double *out, int iters)
{
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
    for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma(double *out, int iters)
{
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[16];
    for (int t = 0; t < 16; ++t) c[t] = t;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 16; ++t) c[t] = fma(a, c[t], b);
    }
    double s = 0; for (int t = 0; t < 16; ++t) s += c[t];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main()
{
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *o; cudaMalloc(&o, 1 << 26);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w : {4, 8, 16}) {
        int iters = 20000;
        dmma<<<sms, 32 * w>>>(o, 10); cudaDeviceSynchronize();
        cudaEventRecord(e0); dmma<<<sms, 32 * w>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 256 * 8 * (double)iters * w * sms;
        printf("DMMA warps/SM %2d: %.2f TFLOP/s\n", w, fl / ms / 1e9);
        cudaEventRecord(e0); dfma<<<sms, 32 * w>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 16 * 32 * (double)iters * w * sms;
        printf("DFMA warps/SM %2d: %.2f TFLOP/s\n", w, fl / ms / 1e9);
    }
    return 0;
}
