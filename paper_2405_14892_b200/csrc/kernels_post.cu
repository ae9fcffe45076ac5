// NEXT-4 — posterior conditioning before Alg. 1 (§V-A, Eq. 7-8):
//   Sigma_post = (Sigma^{-1} + tau^{-2} A^T A)^{-1},  mu_post = mu + tau^{-2} Sigma_post A^T (y - A mu).
// B200 formulation: both are a Schur complement. The augmented symmetric matrix
//        [ Sigma_oo + tau^2 I   Sigma_{o,:}   r ]        r = y - mu_o
//   M =  [ Sigma_{:,o}          Sigma         0 ]
//        [ r^T                  0             1 ]
// factored by the SAME right-looking tiled Cholesky (launch_potrf with ncols = the observation tile
// columns) leaves in its trailing block
//   Sigma - Sigma_{:,o} C^{-1} Sigma_{o,:} = Sigma_post           (Woodbury form of Eq. 7)
//   0 - Sigma_{:,o} C^{-1} r              = -(mu_post - mu)      (Eq. 8)
// so the TRSM (m^2 n) and SYRK (n^2 m) of the conditioning run on the DMMA update kernel. The
// observation block is padded to a tile multiple with decoupled "far" locations (covariance
// exp(-h/beta) underflows to exactly 0), so no special padding logic is needed.
// This file holds the small helpers: diagonal shift, row write / read, diagonal read and the
// symmetric permutation of the Schur complement into sorted order.
#include "common.cuh"
#include "mvn_internal.h"

namespace mvn {

__device__ __forceinline__ int64_t tp_index(int64_t r, int64_t c) {   // element (r, c), r >= c, tile-packed
    return tile_offset(r / kTile, c / kTile) + (c % kTile) * kTile + (r % kTile);
}

__global__ void k_add_diag(double *__restrict__ tiles, int64_t begin, int64_t end, double v) {
    const int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < end) tiles[tp_index(i, i)] += v;
}

__global__ void k_set_row(double *__restrict__ tiles, int64_t row, int64_t col0, int64_t ncols, const double *__restrict__ v) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < ncols) tiles[tp_index(row, col0 + j)] = v[j];
}

// element (rows[j], col0 + j) += v for j < count (rows[j] >= col0 + j): the nugget on the
// site-observation cross covariance of an observed site with its own observation (Cov(x_i, y_j) =
// Sigma_ii = sigma^2 + nugget when i = obs_j, which the Matérn kernel of two distinct indices omits).
__global__ void k_add_pairs(double *__restrict__ tiles, const int64_t *__restrict__ rows, int64_t col0, int64_t count, double v) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < count) tiles[tp_index(rows[j], col0 + j)] += v;
}

__global__ void k_get_row(const double *__restrict__ tiles, int64_t row, int64_t col0, int64_t ncols, double *__restrict__ out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < ncols) out[j] = tiles[tp_index(row, col0 + j)];
}

__global__ void k_get_diag(const double *__restrict__ tiles, int64_t begin, int64_t n, double *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = tiles[tp_index(begin + i, begin + i)];
}

// dst (n x n, tile-packed, lower) = src[off + o(i), off + o(j)] (src tile-packed, lower part read
// symmetrically); dst padding = identity. One CTA per destination tile, threads along columns of
// the tile (each thread walks a column: contiguous destination writes).
__global__ void __launch_bounds__(256) k_permute_sym(const double *__restrict__ src, int64_t off, const int64_t *__restrict__ order,
                                                     int64_t n, double *__restrict__ dst) {
    const int64_t t = blockIdx.x;
    int64_t I = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (I * (I + 1) / 2 > t) --I;
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    const int64_t J = t - I * (I + 1) / 2;
    double *D = dst + tile_offset(I, J);
    for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
        const int c = e / kTile, r = e % kTile;                 // column-major within the tile
        const int64_t gi = I * kTile + r, gj = J * kTile + c;
        double v;
        if (gi >= n || gj >= n) {
            v = (gi == gj) ? 1.0 : 0.0;
        } else if (gi < gj) {
            v = 0.0;                                            // strict upper part of a diagonal tile
        } else {
            int64_t p = off + order[gi], q = off + order[gj];
            if (p < q) { const int64_t x = p; p = q; q = x; }
            v = src[tp_index(p, q)];
        }
        D[e] = v;
    }
}

cudaError_t launch_add_diag(double *tiles, int64_t begin, int64_t end, double v, cudaStream_t st) {
    if (end <= begin) return cudaSuccess;
    k_add_diag<<<(unsigned)((end - begin + 255) / 256), 256, 0, st>>>(tiles, begin, end, v);
    return cudaGetLastError();
}

cudaError_t launch_set_row(double *tiles, int64_t row, int64_t col0, int64_t ncols, const double *v, cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    k_set_row<<<(unsigned)((ncols + 255) / 256), 256, 0, st>>>(tiles, row, col0, ncols, v);
    return cudaGetLastError();
}

cudaError_t launch_add_pairs(double *tiles, const int64_t *rows, int64_t col0, int64_t count, double v, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    k_add_pairs<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(tiles, rows, col0, count, v);
    return cudaGetLastError();
}

cudaError_t launch_get_row(const double *tiles, int64_t row, int64_t col0, int64_t ncols, double *out, cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    k_get_row<<<(unsigned)((ncols + 255) / 256), 256, 0, st>>>(tiles, row, col0, ncols, out);
    return cudaGetLastError();
}

cudaError_t launch_get_diag(const double *tiles, int64_t begin, int64_t n, double *out, cudaStream_t st) {
    k_get_diag<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(tiles, begin, n, out);
    return cudaGetLastError();
}

cudaError_t launch_permute_sym(const double *src, int64_t off, const int64_t *order, int64_t n, double *dst, cudaStream_t st) {
    const int64_t nt = (n + kTile - 1) / kTile;
    k_permute_sym<<<(unsigned)(nt * (nt + 1) / 2), 256, 0, st>>>(src, off, order, n, dst);
    return cudaGetLastError();
}

}  // namespace mvn
