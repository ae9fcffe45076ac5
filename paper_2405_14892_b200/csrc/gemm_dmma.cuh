// Warp-tiled fp64 DMMA GEMM main loop with a cp.async multi-stage shared-memory pipeline.
//
//   acc(BM x BN) += A(BM x K) * B(K x BN)
//
// Both operands are staged "K-major": for each k, BM (resp. BN) consecutive values. This is the
// natural layout of both users:
//   - POTRF trailing update C_ij -= L_ik L_jk^T: a K-chunk of a column-major 128x128 tile is a set
//     of contiguous columns, so A[k][m] = L_ik(m, k) and B[k][n] = L_jk(n, k);
//   - SOV update S_r = L[r-block, 0:r] * Y[0:r, samples]: A from the same tiles, B = the row-major
//     Y history (one row = NB consecutive samples).
// Shared-memory row strides SA, SB are == 4 (mod 16) doubles, so the DMMA fragment loads
// (lane l reads row k = l%4, column l/4) hit 16 distinct 8-byte bank pairs per half-warp.
#pragma once
#include "common.cuh"

namespace mvn {

template <int BK, int SA, int SB, int WM, int WN>
__device__ __forceinline__ void mma_chunk(const double *__restrict__ As, const double *__restrict__ Bs, int wm0,
                                          int wn0, int lane, double (&c)[WM][WN][2]) {
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
        double a[WM], b[WN];
        const int kr = kk + (lane & 3);
#pragma unroll
        for (int i = 0; i < WM; ++i) a[i] = As[kr * SA + wm0 + i * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < WN; ++j) b[j] = Bs[kr * SB + wn0 + j * 8 + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < WM; ++i)
#pragma unroll
            for (int j = 0; j < WN; ++j) dmma(c[i][j][0], c[i][j][1], a[i], b[j]);
    }
}

// Generic pipelined main loop. `load(chunk, stage)` issues the cp.async copies of K-chunk `chunk`
// into pipeline stage `stage` (all threads participate); stage s lives at smemA + s*BK*SA and
// smemB + s*BK*SB.
template <int BK, int STAGES, int SA, int SB, int WM, int WN, typename Loader>
__device__ __forceinline__ void gemm_mainloop(int nchunks, double *smemA, double *smemB, int wm0, int wn0, int lane,
                                              double (&c)[WM][WN][2], Loader &&load) {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nchunks) load(s, s);
        cp_async_commit();
    }
    for (int ch = 0; ch < nchunks; ++ch) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = ch + STAGES - 1;
        if (nxt < nchunks) load(nxt, nxt % STAGES);
        cp_async_commit();
        const int st = ch % STAGES;
        mma_chunk<BK, SA, SB, WM, WN>(smemA + st * BK * SA, smemB + st * BK * SB, wm0, wn0, lane, c);
    }
    cp_async_wait<0>();
    __syncthreads();
}

}  // namespace mvn
