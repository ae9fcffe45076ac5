// K1 — Matérn covariance tile generator (Eq. 6; Alg. 1 line 2) and the
// tile-layout helpers (pack / unpack) plus the small prefix kernels (rescale, finalize).
//
// Layout: lower tile-packed, tile (i,j) i>=j is a 128x128 column-major block at tile_offset(i,j).
// One CTA (256 threads) writes one tile; each thread owns pairs of consecutive rows of a column
// and writes them with one 16-byte store, so a warp writes 512 contiguous bytes per instruction
// (fully coalesced). Locations of the tile's 128 rows and 128 columns are staged in shared memory.
// Bound: HBM stores (8 B per element, 6.4 TB/s -> ~23 fp64-pipe instructions per element at 64
// DFMA/clk/SM) vs the fp64 arithmetic per element: distance (3), sqrt, x = h / beta as a product
// with the host's 1/beta (1; a division costs ~10 plus a slow-path call), exp(-x) with sigma2
// folded in (11, exp_neg_scaled), the nu = 3/2, 5/2 factor (1-2).
#include <math_constants.h>

#include "common.cuh"
#include "mvn_internal.h"

namespace mvn {

// exp(-x) for 0 <= x <= 700 in 11 fp64-pipe instructions (CUDA's exp: ~18 plus branches), with
// the factor sigma2 folded into the table: x = k ln2/32 + r, |r| <= ln2/64, k = round(32 x / ln2)
// (magic-constant rounding), exp(-x) = 2^-(k >> 5) * 2^-((k & 31)/32) * exp(-r); exp(-r) by its
// Taylor polynomial of degree 6 (truncation <= r^7/7! = 3.4e-18 relative), the 32 values
// sigma2 * 2^-(j/32) from a host table (long double, correctly rounded), and 2^-(k >> 5) applied
// to the exponent field with an integer subtract (INT pipe). Error <= ~3 ulp (vs ~1 for exp()).
struct MaternArgs {
    int64_t n;
    const double *xy;
    double sigma2, inv_beta, nugget;
    double *tiles;
    double tab[32];      // sigma2 * 2^(-j/32), j = 0..31
};

__device__ __forceinline__ double exp_neg_scaled(double x, const double *tb) {
    constexpr double kMagic = 0x1.8p52;                   // 1.5 * 2^52: fma(.., .., kMagic) rounds to an integer
    constexpr double k32ln2 = 46.166241308446828384;      // 32 / ln 2
    constexpr double kLn2hi = 0x1.62e42fefa3800p-6;       // ln2/32, high part (exact product with k < 2^20)
    constexpr double kLn2lo = 0x1.ef35793c76730p-50;      // ln2/32 - kLn2hi (rounded)
    const double kd = fma(x, k32ln2, kMagic);
    const int k = __double2loint(kd);
    const double kf = kd - kMagic;
    double r = fma(-kf, kLn2hi, x);
    r = fma(-kf, kLn2lo, r);
    double p = 1.0 / 720.0;                               // exp(-r) = sum (-r)^i / i!
    p = fma(p, r, -1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, -1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, -1.0);
    p = fma(p, r, 1.0);
    const double v = tb[k & 31] * p;
    return __hiloint2double(__double2hiint(v) - ((k >> 5) << 20), __double2loint(v));
}

static __device__ __noinline__ double exp_neg_far(double x, double sigma2) { return sigma2 * exp(-x); }

template <int NU2>  // 2*nu: 1 -> nu = 1/2, 3 -> nu = 3/2, 5 -> nu = 5/2; returns sigma2 * C(x)
__device__ __forceinline__ double matern_scaled(double x, double sigma2, const double *tb) {
    const double e = x <= 700.0 ? exp_neg_scaled(x, tb) : exp_neg_far(x, sigma2);   // far pairs: libm path
    if (NU2 == 1) return e;
    if (NU2 == 3) return fma(x, e, e);
    return fma(fma(x, 1.0 / 3.0, 1.0) * x, e, e);
}

template <int NU2>
__global__ void __launch_bounds__(256) k_cov_matern(const MaternArgs p) {
    __shared__ double rx[kTile], ry[kTile], cx[kTile], cy[kTile], tb[32];
    // blockIdx.x -> tile (ti, tj), ti >= tj, row-major enumeration of the lower triangle
    const int64_t id = blockIdx.x;
    int ti = (int)((sqrt(8.0 * (double)id + 1.0) - 1.0) * 0.5);
    while ((int64_t)ti * (ti + 1) / 2 > id) --ti;
    while ((int64_t)(ti + 1) * (ti + 2) / 2 <= id) ++ti;
    const int tj = (int)(id - (int64_t)ti * (ti + 1) / 2);
    const int tid = threadIdx.x;
    const int64_t n = p.n;
    if (tid < kTile) {
        int64_t r = (int64_t)ti * kTile + tid;
        rx[tid] = r < n ? p.xy[2 * r] : 0.0;
        ry[tid] = r < n ? p.xy[2 * r + 1] : 0.0;
    } else {
        int64_t c = (int64_t)tj * kTile + (tid - kTile);
        cx[tid - kTile] = c < n ? p.xy[2 * c] : 0.0;
        cy[tid - kTile] = c < n ? p.xy[2 * c + 1] : 0.0;
    }
    if (tid < 32) tb[tid] = p.tab[tid];
    __syncthreads();
    double *T = p.tiles + tile_offset(ti, tj);
    const int64_t r0 = (int64_t)ti * kTile, c0 = (int64_t)tj * kTile;
    const bool edge = r0 + kTile > n || ti == tj;         // padding or diagonal elements in this tile
    const double sigma2 = p.sigma2, ib = p.inv_beta, diag = p.sigma2 + p.nugget;
    // 128 columns x 64 row-pairs = 8192 double2 stores; 256 threads -> 32 each (a warp stores 512
    // contiguous bytes per instruction)
#pragma unroll 4
    for (int it = 0; it < 32; ++it) {
        const int e = it * 256 + tid;
        const int col = e >> 6;
        const int rp = (e & 63) * 2;
        double v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int row = rp + h;
            const double dx = rx[row] - cx[col];
            const double dy = ry[row] - cy[col];
            double val = matern_scaled<NU2>(sqrt(fma(dx, dx, dy * dy)) * ib, sigma2, tb);
            if (edge) {
                const int64_t gr = r0 + row, gc = c0 + col;
                if (gr >= n || gc >= n) val = (gr == gc) ? 1.0 : 0.0;
                else if (gr == gc) val = diag;
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
    MaternArgs a;
    a.n = n; a.xy = xy; a.sigma2 = sigma2; a.inv_beta = 1.0 / beta; a.nugget = nugget; a.tiles = tiles;
    for (int j = 0; j < 32; ++j) a.tab[j] = (double)((long double)sigma2 * exp2l(-(long double)j / 32.0L));
    dim3 grid((unsigned)ntiles);
    if (nu == 0.5) k_cov_matern<1><<<grid, 256, 0, st>>>(a);
    else if (nu == 1.5) k_cov_matern<3><<<grid, 256, 0, st>>>(a);
    else k_cov_matern<5><<<grid, 256, 0, st>>>(a);
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
