// K1 — Matérn covariance tile generator (Eq. 6; Alg. 1 line 2) and the
// tile-layout helpers (pack / unpack) plus the small prefix kernels (rescale, finalize).
//
// Layout: lower tile-packed, tile (i,j) i>=j is a 128x128 column-major block at tile_offset(i,j).
// One CTA (256 threads) writes one tile (layout in k_cov_matern's header); every store is part of
// a warp-wide 1 KB contiguous column write.
// Bound: HBM stores (8 B per element, 6.4 TB/s -> ~23 fp64-pipe instructions per element at 64
// DFMA/clk/SM) vs the fp64 arithmetic per element: distance (3), sqrt, x = h / beta as a product
// with the host's 1/beta (1; a division costs ~10 plus a slow-path call), exp(-x) with sigma2
// folded in (8, exp_neg_scaled), the nu = 3/2, 5/2 factor (1-2).
#include <cstdlib>

#include <math_constants.h>

#include "common.cuh"
#include "mvn_internal.h"

namespace mvn {

// exp(-x) for 0 <= x <= 700 in 8 fp64-pipe instructions (CUDA's exp: ~18 plus branches), with
// the factor sigma2 folded into the table: x = k ln2/1024 + r, |r| <= ln2/2048, k = round(1024 x / ln2)
// (magic-constant rounding), exp(-x) = 2^-(k >> 10) * 2^-((k & 1023)/1024) * exp(-r); exp(-r) by its
// Taylor polynomial of degree 3 (truncation <= r^4/4! = 5.5e-16 relative), the 1,024 values
// sigma2 * 2^-(j/1024) in shared memory (2^-(j/1024) correctly rounded on the host once per context,
// g_exp2n, times sigma2 per CTA), and 2^-(k >> 10) applied to the exponent field with an integer
// subtract. Error <= ~5 ulp (round 2, session 2: one fp64 FMA fewer than the 256-entry, degree-4 form).
struct MaternArgs {
    int64_t n;
    const double *xy;
    double sigma2, inv_beta, nugget;
    TileMap tm;          // destination storage (the full buffer, or a rank's owned tile columns)
    int libm;            // sigma2 so small or large that the scaled result could leave the normal range
};

__device__ double g_exp2n[1024];   // 2^(-j/1024), j = 0..1023 (matern_init)

__device__ __forceinline__ double exp_neg_scaled(double x, const double *tb) {
    constexpr double kMagic = 0x1.8p52;                   // 1.5 * 2^52: fma(.., .., kMagic) rounds to an integer
    constexpr double k1024ln2 = 1477.3197218702985;       // 1024 / ln 2
    constexpr double kLn2hi = 0x1.62e42fefa2000p-11;      // ln2/1024, high part (40 bits)
    constexpr double kLn2lo = 0x1.9ef35793c7673p-51;      // ln2/1024 - kLn2hi (rounded)
    const double kd = fma(x, k1024ln2, kMagic);
    const int k = __double2loint(kd);
    const double kf = kd - kMagic;
    double r = fma(-kf, kLn2hi, x);
    r = fma(-kf, kLn2lo, r);
    double p = -1.0 / 6.0;                                // exp(-r) = sum (-r)^i / i!
    p = fma(p, r, 0.5);
    p = fma(p, r, -1.0);
    p = fma(p, r, 1.0);
    const double v = tb[k & 1023] * p;
    return __hiloint2double(__double2hiint(v) - ((k >> 10) << 20), __double2loint(v));
}

template <int NU2>  // 2*nu: 1 -> nu = 1/2, 3 -> nu = 3/2, 5 -> nu = 5/2; sigma2 * C(x) from e = sigma2 exp(-x)
__device__ __forceinline__ double matern_poly(double x, double e) {
    if (NU2 == 1) return e;
    if (NU2 == 3) return fma(x, e, e);
    return fma(fma(x, 1.0 / 3.0, 1.0) * x, e, e);
}

// The tiles with far pairs (x > 699): libm's sqrt and exp, out of line (keeps the fast path's
// register budget).
template <int NU2>
static __device__ __noinline__ double matern_far(double d2, double ib, double sigma2) {
    const double x = sqrt(d2) * ib;
    return matern_poly<NU2>(x, sigma2 * exp(-x));
}

// sqrt(d) for d >= 1e-300 (the caller adds 1e-300 to the squared distance inside its last FMA, so
// coincident points give 1e-150 and C = sigma2 exactly, and no special-operand branch is needed):
// the MUFU reciprocal square-root seed, one coupled (Goldschmidt) step on t ~ sqrt(d) and
// h ~ 1 / (2 sqrt(d)) — the seed's relative error squares — then one Newton correction of t
// (correctly rounded in an exact-arithmetic emulation with seed errors up to 2^-21). 2 DMUL + 5 DFMA;
// the d + 1e-300 add and the separate rsqrt refinement of the previous version cost 3 more fp64
// instructions per element (22 instead of 25; K1 at D 4.07-4.11 -> 3.83-3.94 ms).
__device__ __forceinline__ double sqrt_pos(double d) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double t = d * y, h = 0.5 * y;
    const double r = fma(-t, h, 0.5);
    t = fma(t, r, t);
    h = fma(h, r, h);
    return fma(h, fma(-t, t, d), t);
}

// One CTA (256 threads) per tile. Thread t owns RPT consecutive rows of the tile (their locations in
// registers; RPT = 4: rows 4 (t % 32) .., the columns t / 32 + 8 m; RPT = 8: rows 8 (t % 16) .., the
// columns t / 16 + 16 m): per column RPT / 2 16-byte stores, so each group of 128 / RPT lanes writes
// one whole 1 KB column (coalesced), and a column's location is one shared-memory read for RPT
// elements. The libm fallback for far pairs (x > 699, where sigma2 e^-x nears the bottom of the
// normal range) is decided once per tile from the bounding boxes of its row and column locations.
template <int NU2, int RPT, int MINB>
__global__ void __launch_bounds__(256, MINB) k_cov_matern(const MaternArgs p) {
    constexpr int TPC = kTile / RPT;                     // threads per column
    constexpr int CPI = 256 / TPC;                       // columns per step
    __shared__ double cx[kTile], cy[kTile], rxs[kTile], rys[kTile], tb[1024], bb[8][4];
    __shared__ int fast_s;
    // blockIdx.x -> tile (ti, tj), ti >= tj, row-major enumeration of the lower triangle
    const int64_t id = blockIdx.x;
    int ti = (int)((sqrt(8.0 * (double)id + 1.0) - 1.0) * 0.5);
    while ((int64_t)ti * (ti + 1) / 2 > id) --ti;
    while ((int64_t)(ti + 1) * (ti + 2) / 2 <= id) ++ti;
    const int tj = (int)(id - (int64_t)ti * (ti + 1) / 2);
    if (!p.tm.owns_col(tj) || !p.tm.owns_row(ti)) return;   // distributed storage: another rank's tile
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = p.n;
    const int64_t r0 = (int64_t)ti * kTile, c0 = (int64_t)tj * kTile;
    double vx, vy;                                       // this thread's location (column, then row)
    if (tid < kTile) {
        const int64_t c = c0 + tid;
        vx = c < n ? p.xy[2 * c] : p.xy[2 * c0];        // padding: a real location of the block
        vy = c < n ? p.xy[2 * c + 1] : p.xy[2 * c0 + 1];
        cx[tid] = vx;
        cy[tid] = vy;
    } else {
        const int64_t r = r0 + tid - kTile;
        vx = r < n ? p.xy[2 * r] : p.xy[2 * r0];
        vy = r < n ? p.xy[2 * r + 1] : p.xy[2 * r0 + 1];
        rxs[tid - kTile] = vx;
        rys[tid - kTile] = vy;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) tb[tid + 256 * q] = p.sigma2 * g_exp2n[tid + 256 * q];
    {   // bounding boxes: warps 0-3 the columns, warps 4-7 the rows
        double mnx = vx, mxx = vx, mny = vy, mxy = vy;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mnx = fmin(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
            mxx = fmax(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
            mny = fmin(mny, __shfl_xor_sync(0xffffffffu, mny, o));
            mxy = fmax(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
        }
        if (lane == 0) { bb[warp][0] = mnx; bb[warp][1] = mxx; bb[warp][2] = mny; bb[warp][3] = mxy; }
    }
    __syncthreads();
    if (tid == 0) {
        double b[2][4];
        for (int h = 0; h < 2; ++h) {
            b[h][0] = bb[4 * h][0]; b[h][1] = bb[4 * h][1]; b[h][2] = bb[4 * h][2]; b[h][3] = bb[4 * h][3];
            for (int w = 4 * h + 1; w < 4 * h + 4; ++w) {
                b[h][0] = fmin(b[h][0], bb[w][0]); b[h][1] = fmax(b[h][1], bb[w][1]);
                b[h][2] = fmin(b[h][2], bb[w][2]); b[h][3] = fmax(b[h][3], bb[w][3]);
            }
        }
        const double ex = fmax(b[0][1] - b[1][0], b[1][1] - b[0][0]), ey = fmax(b[0][3] - b[1][2], b[1][3] - b[0][2]);
        fast_s = !p.libm && sqrt(ex * ex + ey * ey) * p.inv_beta <= 699.0;
    }
    const int rq = (tid % TPC) * RPT, cg = tid / TPC;
    __syncthreads();
    double rx[RPT], ry[RPT];
#pragma unroll
    for (int h = 0; h < RPT; ++h) { rx[h] = rxs[rq + h]; ry[h] = rys[rq + h]; }
    double *T = p.tm.tile(ti, tj) + rq;
    const bool edge = r0 + kTile > n || ti == tj;         // padding or diagonal elements in this tile
    const double sigma2 = p.sigma2, ib = p.inv_beta, diag = p.sigma2 + p.nugget;
    const bool fast = fast_s != 0;
#pragma unroll 1
    for (int m = 0; m < kTile / CPI; ++m) {
        const int col = cg + CPI * m;
        const double xc = cx[col], yc = cy[col];
        double v[RPT];
        if (fast) {
#pragma unroll
            for (int h = 0; h < RPT; ++h) {
                const double dx = rx[h] - xc, dy = ry[h] - yc;
                const double x = sqrt_pos(fma(dx, dx, fma(dy, dy, 1e-300))) * ib;
                v[h] = matern_poly<NU2>(x, exp_neg_scaled(x, tb));
            }
        } else {
#pragma unroll
            for (int h = 0; h < RPT; ++h) {
                const double dx = rx[h] - xc, dy = ry[h] - yc;
                v[h] = matern_far<NU2>(fma(dx, dx, dy * dy), ib, sigma2);
            }
        }
        if (edge) {
#pragma unroll
            for (int h = 0; h < RPT; ++h) {
                const int64_t gr = r0 + rq + h, gc = c0 + col;
                if (gr >= n || gc >= n) v[h] = (gr == gc) ? 1.0 : 0.0;
                else if (gr == gc) v[h] = diag;
            }
        }
        double2 *dst = reinterpret_cast<double2 *>(T + (int64_t)col * kTile);
#pragma unroll
        for (int h = 0; h < RPT / 2; ++h) dst[h] = make_double2(v[2 * h], v[2 * h + 1]);
    }
}

// variant (rows per thread, CTAs per SM): MVN_K1_VARIANT = 0 (4, 4: default), 1 (4, 5), 2 (2, 6),
// 3 (2, 8), 4 (8, 4) — an experiment knob read once
static int k1_variant() {
    static const int v = [] { const char *e = getenv("MVN_K1_VARIANT"); const int x = e ? atoi(e) : 0; return x >= 0 && x <= 4 ? x : 0; }();
    return v;
}

template <int NU2>
static void k1_launch(dim3 grid, const MaternArgs &a, cudaStream_t st) {
    switch (k1_variant()) {
        case 1: k_cov_matern<NU2, 4, 5><<<grid, 256, 0, st>>>(a); break;
        case 2: k_cov_matern<NU2, 2, 6><<<grid, 256, 0, st>>>(a); break;
        case 3: k_cov_matern<NU2, 2, 8><<<grid, 256, 0, st>>>(a); break;
        case 4: k_cov_matern<NU2, 8, 4><<<grid, 256, 0, st>>>(a); break;
        default: k_cov_matern<NU2, 4, 4><<<grid, 256, 0, st>>>(a); break;
    }
}

cudaError_t matern_init() {
    static double h[1024];
    for (int j = 0; j < 1024; ++j) h[j] = (double)exp2l(-(long double)j / 1024.0L);
    return cudaMemcpyToSymbol(g_exp2n, h, sizeof(h));
}

cudaError_t launch_cov_matern_map(int64_t n, const double *xy, double sigma2, double beta, double nu, double nugget,
                                  const TileMap &tm, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int64_t ntiles = (int64_t)nt * (nt + 1) / 2;
    MaternArgs a;
    a.n = n; a.xy = xy; a.sigma2 = sigma2; a.inv_beta = 1.0 / beta; a.nugget = nugget; a.tm = tm;
    a.libm = sigma2 < 0x1p-100 || sigma2 > 0x1p100;
    dim3 grid((unsigned)ntiles);
    if (nu == 0.5) k1_launch<1>(grid, a, st);
    else if (nu == 1.5) k1_launch<3>(grid, a, st);
    else k1_launch<5>(grid, a, st);
    return cudaGetLastError();
}

cudaError_t launch_cov_matern(int64_t n, const double *xy, double sigma2, double beta, double nu, double nugget,
                              double *tiles, cudaStream_t st) {
    return launch_cov_matern_map(n, xy, sigma2, beta, nu, nugget, TileMap::full(tiles), st);
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
