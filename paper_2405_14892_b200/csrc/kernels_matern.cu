// K1 — Matérn covariance tile generator (Eq. 6; Alg. 1 line 2) and the
// tile-layout helpers (pack / unpack) plus the small prefix kernels (rescale, finalize).
//
// Layout: lower tile-packed, tile (i,j) i>=j is a 128x128 column-major block at tile_offset(i,j).
// One CTA (256 threads) writes one tile; each thread owns pairs of consecutive rows of a column
// and writes them with one 16-byte store, so a warp writes 512 contiguous bytes per instruction
// (fully coalesced). Locations of the tile's 128 rows and 128 columns are staged in shared memory.
// Bound: HBM stores (8 B per element) vs fp64 exp (~20 DFMA-pipe instructions per element).
#include <math_constants.h>

#include "common.cuh"
#include "mvn_internal.h"

namespace mvn {

template <int NU2>  // 2*nu: 1 -> nu = 1/2, 3 -> nu = 3/2, 5 -> nu = 5/2
__device__ __forceinline__ double matern_half(double x) {
    const double e = exp(-x);
    if (NU2 == 1) return e;
    if (NU2 == 3) return (1.0 + x) * e;
    return (1.0 + x + x * x * (1.0 / 3.0)) * e;
}

template <int NU2>
__global__ void __launch_bounds__(256) k_cov_matern(int64_t n, int nt, const double *__restrict__ xy,
                                                   double sigma2, double beta, double nugget,
                                                   double *__restrict__ tiles) {
    __shared__ double rx[kTile], ry[kTile], cx[kTile], cy[kTile];
    // blockIdx.x -> tile (ti, tj), ti >= tj, row-major enumeration of the lower triangle
    const int64_t id = blockIdx.x;
    int ti = (int)((sqrt(8.0 * (double)id + 1.0) - 1.0) * 0.5);
    while ((int64_t)ti * (ti + 1) / 2 > id) --ti;
    while ((int64_t)(ti + 1) * (ti + 2) / 2 <= id) ++ti;
    const int tj = (int)(id - (int64_t)ti * (ti + 1) / 2);
    const int tid = threadIdx.x;
    if (tid < kTile) {
        int64_t r = (int64_t)ti * kTile + tid;
        rx[tid] = r < n ? xy[2 * r] : 0.0;
        ry[tid] = r < n ? xy[2 * r + 1] : 0.0;
    } else {
        int64_t c = (int64_t)tj * kTile + (tid - kTile);
        cx[tid - kTile] = c < n ? xy[2 * c] : 0.0;
        cy[tid - kTile] = c < n ? xy[2 * c + 1] : 0.0;
    }
    __syncthreads();
    double *T = tiles + tile_offset(ti, tj);
    const int64_t r0 = (int64_t)ti * kTile, c0 = (int64_t)tj * kTile;
    // 128 columns x 64 row-pairs = 8192 double2 stores; 256 threads -> 32 each
#pragma unroll 4
    for (int it = 0; it < 32; ++it) {
        const int e = it * 256 + tid;
        const int col = e >> 6;
        const int rp = (e & 63) * 2;
        double v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int row = rp + h;
            const int64_t gr = r0 + row, gc = c0 + col;
            double val;
            if (gr >= n || gc >= n) {
                val = (gr == gc) ? 1.0 : 0.0;
            } else if (gr == gc) {
                val = sigma2 + nugget;
            } else {
                const double dx = rx[row] - cx[col];
                const double dy = ry[row] - cy[col];
                const double hh = sqrt(dx * dx + dy * dy);
                val = sigma2 * matern_half<NU2>(hh / beta);
            }
            v[h] = val;
        }
        *reinterpret_cast<double2 *>(T + (int64_t)col * kTile + rp) = make_double2(v[0], v[1]);
    }
}

cudaError_t launch_cov_matern(int64_t n, const double *xy, double sigma2, double beta, double nu, double nugget,
                              double *tiles, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int64_t ntiles = (int64_t)nt * (nt + 1) / 2;
    dim3 grid((unsigned)ntiles);
    if (nu == 0.5) k_cov_matern<1><<<grid, 256, 0, st>>>(n, nt, xy, sigma2, beta, nugget, tiles);
    else if (nu == 1.5) k_cov_matern<3><<<grid, 256, 0, st>>>(n, nt, xy, sigma2, beta, nugget, tiles);
    else k_cov_matern<5><<<grid, 256, 0, st>>>(n, nt, xy, sigma2, beta, nugget, tiles);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ pack / unpack
__global__ void k_pack(int64_t n, double *__restrict__ dense, int64_t ld, double *__restrict__ tiles, int to_tiles) {
    const int64_t id = blockIdx.x;
    int ti = (int)((sqrt(8.0 * (double)id + 1.0) - 1.0) * 0.5);
    while ((int64_t)ti * (ti + 1) / 2 > id) --ti;
    while ((int64_t)(ti + 1) * (ti + 2) / 2 <= id) ++ti;
    const int tj = (int)(id - (int64_t)ti * (ti + 1) / 2);
    double *T = tiles + tile_offset(ti, tj);
    for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
        const int col = e / kTile, row = e % kTile;
        const int64_t gr = (int64_t)ti * kTile + row, gc = (int64_t)tj * kTile + col;
        const bool inside = gr < n && gc < n;
        if (to_tiles) {
            double v;
            if (!inside) v = (gr == gc) ? 1.0 : 0.0;
            else if (gr >= gc) v = dense[gc * ld + gr];
            else v = dense[gr * ld + gc];   // upper part of a diagonal tile: mirror (symmetric)
            T[e] = v;
        } else if (inside) {
            if (gr >= gc) {
                dense[gc * ld + gr] = T[e];
                if (gr != gc) dense[gr * ld + gc] = 0.0;
            }
        }
    }
}

cudaError_t launch_pack(int64_t n, const double *dense, int64_t ld, double *tiles, bool to_tiles, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int64_t ntiles = (int64_t)nt * (nt + 1) / 2;
    k_pack<<<(unsigned)ntiles, 256, 0, st>>>(n, const_cast<double *>(dense), ld, tiles, to_tiles ? 1 : 0);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ prefix helpers
__global__ void k_rescale(int64_t n, const double *__restrict__ Mg, double *__restrict__ M, double *__restrict__ S) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double m = M[k], mg = Mg[k];
    S[k] = (m == -CUDART_INF) ? 0.0 : S[k] * exp(m - mg);
    M[k] = mg;
}

__global__ void k_finalize(int64_t n, double lognr, const double *__restrict__ M, const double *__restrict__ S,
                           double *__restrict__ logP) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double s = S[k];
    logP[k] = (s > 0.0) ? M[k] + log(s) - lognr : -CUDART_INF;
}

// Limits check for mvn_sov_prefix: flag = 1 if any a_k or b_k is NaN or a_k > b_k (b = NULL: +inf).
__global__ void k_check_limits(int64_t n, const double *__restrict__ a, const double *__restrict__ b, int *__restrict__ flag) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double ak = a[k];
    const double bk = b ? b[k] : CUDART_INF;
    if (isnan(ak) || isnan(bk) || ak > bk) atomicOr(flag, 1);
}

cudaError_t launch_check_limits(int64_t n, const double *a, const double *b, int *flag, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    k_check_limits<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, a, b, flag);
    return cudaGetLastError();
}

cudaError_t launch_rescale(int64_t n, const double *Mg, double *M, double *S, cudaStream_t st) {
    k_rescale<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, Mg, M, S);
    return cudaGetLastError();
}
cudaError_t launch_finalize(int64_t n, int64_t NR, const double *M, const double *S, double *logP, cudaStream_t st) {
    k_finalize<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, log((double)NR), M, S, logP);
    return cudaGetLastError();
}

}  // namespace mvn
