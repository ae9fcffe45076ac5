// Micro-benchmark (tooling): latency of one SOV chain step (normal.cuh) per row, for chain warps
// alone and next to warps that saturate the fp64 tensor pipe with DMMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2405_14892_b200/csrc/common.cuh"
#include "../paper_2405_14892_b200/csrc/normal.cuh"

using namespace mvn;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_chain(int rows, int nchain, int ndmma, long long *cyc, double *sink) {
    const int warp = threadIdx.x >> 5;
    if (warp < nchain) {
        double s = 0.1 * threadIdx.x, ell = 0.0;
        const uint64_t G = 0x6A09E667F3BCC908ull;
        long long t0 = clock64();
        for (int k = 0; k < rows; ++k) {
            const double ap = (-0.3 - s) * 1.7;
            const uint64_t X = (uint64_t)(threadIdx.x + 1) * G + mix(0x1234ull + k);
            const double w = ((double)(X >> 12) + 0.5) * 0x1p-52;
            double lq, y;
            double qq;
            sov_step_upper(ap, w, lq, y, qq);
            ell += lq;
            s = 0.5 * s + 0.3 * y;           // next row depends on this y (like the in-block dot)
        }
        long long t1 = clock64();
        if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / rows;
        if (ell == 1.2345) sink[0] = ell + s;
    } else if (warp < nchain + ndmma) {
        double c[8][2] = {};
        double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
        for (int it = 0; it < rows * 40; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
        double t = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) t += c[i][0] + c[i][1];
        if (t == 1.2345) sink[0] = t;
    }
}

int main() {
    long long *cyc; double *sink;
    cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 8);
    for (int nchain : {1, 4}) {
        for (int ndmma : {0, 8}) {
            const int rows = 512;
            k_chain<<<148, 32 * (nchain + ndmma)>>>(rows, nchain, ndmma, cyc, sink);
            cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            printf("{\"chain_warps\":%d,\"dmma_warps\":%d,\"cycles_per_row\":%lld}\n", nchain, ndmma, h[0]);
        }
    }
    printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
