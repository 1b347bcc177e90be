// K4 probe: cycles of the one-warp FGS body (k4_small.cuh) on a synthetic
// s x s Gram block, measured inside one kernel with clock64 (no launch
// overhead): total per call, at nu = 1 (mostly the fixed part) and nu = 25.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2512_09642_b200/csrc \
//        -I include -o /tmp/k4_probe tools/k4_probe.cu && /tmp/k4_probe
#include <cstdio>
#include <vector>
#include <cmath>

#include "k4_small.cuh"

using namespace sscg;

template <int NB4>
__global__ void probe(K4Args a, DevState *st, long long *cyc, int reps)
{
    __shared__ double scratch[32 * 32 + 32 + 64];
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x == 0) { st->k = 0; st->done = 0; }
        __syncwarp();
        k4_fgs_small<NB4>(a, st, scratch);
        __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = (t1 - t0) / reps;
}

int main()
{
    for (int s : {8, 16}) {
        for (int nu : {1, 25}) {
            const int nent = s * s + s;
            std::vector<double> h(nent);
            // Ghat = Gram of s smooth-ish vectors (SPD), c = first column
            for (int i = 0; i < s; ++i)
                for (int j = 0; j < s; ++j) h[i * s + j] = 1.0 / (1.0 + std::fabs(i - j)) + (i == j ? 1.0 : 0.0);
            for (int i = 0; i < s; ++i) h[s * s + i] = h[i * s];
            double *blk, *buf;
            DevState *st;
            long long *cyc;
            cudaMalloc(&blk, nent * 8);
            cudaMalloc(&buf, 1 << 20);
            cudaMalloc(&st, sizeof(DevState));
            cudaMalloc(&cyc, 8);
            cudaMemcpy(blk, h.data(), nent * 8, cudaMemcpyHostToDevice);
            DevState hs{};
            hs.hist_cap = 4;
            hs.gram_cap = 4;
            hs.rtol = 0.0;
            hs.max_outer = 1 << 20;
            cudaMemcpy(st, &hs, sizeof hs, cudaMemcpyHostToDevice);
            K4Args a{};
            a.blk = blk;
            a.alpha = buf;
            a.s = s;
            a.nu = nu;
            a.h_gram = buf + 1024; a.h_d = buf + 8192; a.h_at = buf + 9000; a.h_al = buf + 10000;
            a.h_delta = buf + 11000; a.h_relres = buf + 12000; a.h_lnorm = buf + 13000;
            long long c0 = 0;
            if (s == 8) probe<2><<<1, 32>>>(a, st, cyc, 200);
            else probe<4><<<1, 32>>>(a, st, cyc, 200);
            cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
            printf("s=%2d nu=%2d  %7lld cycles per call\n", s, nu, c0);
            cudaFree(blk); cudaFree(buf); cudaFree(st); cudaFree(cyc);
        }
    }
    return cudaGetLastError() != cudaSuccess;
}
