// TMA element-stride probe (sm_100a): how many elements does a tiled load with
// elementStrides[0] = 2 deliver, and where?  A 2-D tensor [8 rows][64 cols]
// (value = 1000*row + col), box {16, 2}, element stride {2, 1}.  The mbarrier
// wait is bounded (no hang if the byte count is wrong).  Measured on a B200
// (profiles/r02g_tma_stride_probe.txt): all 16 contiguous elements of each row
// arrive -- the innermost element stride does not subsample, so an even/odd
// split of the K1M stage cannot come from two strided TMA loads.  (A box start
// at an odd element raised "illegal instruction"; only x0 = 0 is run here.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma_stride tools/tma_stride_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

__global__ void probe(const __grid_constant__ CUtensorMap m, int x0, unsigned expect, double *out, int *ok)
{
    __shared__ alignas(128) double box[64];
    __shared__ alignas(8) unsigned long long bar;
    for (int i = threadIdx.x; i < 64; i += blockDim.x) box[i] = -1.0;
    __syncthreads();
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar), d = (unsigned)__cvta_generic_to_shared(box);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(expect));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(d), "l"(&m), "r"(x0), "r"(0), "r"(b) : "memory");
        int done = 0;
        for (long it = 0; it < 20000000 && !done; ++it) {
            unsigned r;
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(r) : "r"(b));
            done = r;
        }
        *ok = done;
        for (int i = 0; i < 64; ++i) out[i] = box[i];
    }
}

int main()
{
    double h[8 * 64];
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 64; ++c) h[r * 64 + c] = 1000.0 * r + c;
    double *g, *out;
    int *ok;
    cudaMalloc(&g, sizeof h);
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMalloc(&ok, sizeof(int));
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    CUtensorMap m;
    cuuint64_t dims[2] = {64, 8};
    cuuint64_t strides[1] = {64 * 8};
    cuuint32_t box[2] = {16, 2}, es[2] = {2, 1};
    CUresult rc = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, strides, box, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc = %d\n", (int)rc);
    for (int x0 : {0}) {
        for (unsigned expect : {32u * 8u}) {   // 16 elements x 2 rows (the larger count first: a shortfall only times out)
            probe<<<1, 32>>>(m, x0, expect, out, ok);
            cudaError_t e = cudaDeviceSynchronize();
            double o[64];
            int k = 0;
            cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost);
            cudaMemcpy(&k, ok, sizeof k, cudaMemcpyDeviceToHost);
            printf("x0=%d expect=%u bytes: completed=%d err=%s\n  ", x0, expect, k, cudaGetErrorString(e));
            for (int i = 0; i < 34; ++i) printf("%g ", o[i]);
            printf("\n");
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
