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
#include <cmath>
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
// General nu (Eq. 6 with any nu > 0; P:446's wind fit has nu = 1.43391): K_nu(x) by Temme's method —
// nu = nl + mu, |mu| <= 1/2: for x <= 2 Temme's series for K_mu and K_mu+1, for x > 2 Steed's
// continued fraction CF2 (Thompson-Barnett form) — then the forward recurrence
// K_{mu+i+1} = 2 (mu+i)/x K_{mu+i} + K_{mu+i-1} (stable for K). Everything that depends on nu only is
// computed on the host in long double (the Gamma-function terms, mu pi / sin(mu pi), and the
// reciprocals of the iterations' denominators), so a Temme step has no division and a CF2 step one.
namespace matg {
constexpr int TMAX = 32, CMAX = 112;  // Temme / CF2 caps (x <= 2: c_k <= 1/k!^2 -> 1e-30 by k = 18; CF2 just above x = 2 needs ~100: 64 left 2e-14)
}
struct MaternGen {
    double mu, fact, gam1, gam2, gp, gm, pref;         // gp, gm = Gamma(1 + mu), Gamma(1 - mu); pref = 2^(1-nu) / Gamma(nu)
    int nl;
    double rq[matg::TMAX], rim[matg::TMAX], rip[matg::TMAX];   // 1/(k^2 - mu^2), 1/(k - mu), 1/(k + mu), k >= 1
    double ria[matg::CMAX], rinv[matg::CMAX];                  // CF2: 1/a_i (a_i = -(1/4 - mu^2) - i(i-1)), 1/i
};

struct MaternArgs {
    int64_t n;
    const double *xy;
    double sigma2, inv_beta, nugget;
    TileMap tm;          // destination storage (the full buffer, or a rank's owned tile columns)
    int libm;            // sigma2 so small or large that the scaled result could leave the normal range
    MaternGen gen;       // general nu only
};

// sigma2 * 2^(1-nu)/Gamma(nu) * x^nu * K_nu(x), x > 0 (Eq. 6)
__device__ __forceinline__ double matern_general(double x, double sigma2, const MaternGen &g) {
    if (x < 1e-100) return sigma2;                        // coincident points: the limit sigma2
    const double mu = g.mu, mu2 = mu * mu;
    double kmu, k1;
    if (x <= 2.0) {
        const double x2 = 0.5 * x, d = -log(x2);          // d = ln(2/x)
        const double e = mu * d;
        const double E = exp(e), Ei = 1.0 / E;
        const double ch = 0.5 * (E + Ei), sh_e = e == 0.0 ? 1.0 : sinh(e) / e;   // (E - 1/E) / 2e would cancel for small e
        double ff = g.fact * (g.gam1 * ch + g.gam2 * sh_e * d);
        double p = 0.5 * E * g.gp;                        // 0.5 (x/2)^-mu Gamma(1 + mu)
        double q = 0.5 * Ei * g.gm;                       // 0.5 (x/2)^mu Gamma(1 - mu)
        double c = 1.0, sum = ff, sum1 = p;
        const double dd = x2 * x2;
        for (int k = 1; k < matg::TMAX; ++k) {
            ff = (k * ff + p + q) * g.rq[k];
            c *= dd * g.rinv[k];
            p *= g.rim[k];
            q *= g.rip[k];
            const double del = c * ff;
            sum += del;
            sum1 += c * (p - k * ff);
            if (fabs(del) < fabs(sum) * 1e-17) break;
        }
        kmu = sum;
        k1 = sum1 * (2.0 / x);
    } else {
        double b = 2.0 * (1.0 + x), d = 1.0 / b, h = d, delh = d, q1 = 0.0, q2 = 1.0;
        const double a1 = 0.25 - mu2;
        double q = a1, c = a1, a = -a1, s = 1.0 + q * delh;
        for (int i = 2; i < matg::CMAX; ++i) {
            a -= 2 * (i - 1);
            c = -a * c * g.rinv[i];
            const double qnew = (q1 - b * q2) * g.ria[i];
            q1 = q2;
            q2 = qnew;
            q += c * qnew;
            b += 2.0;
            d = 1.0 / (b + a * d);
            delh = (b * d - 1.0) * delh;
            h += delh;
            const double dels = q * delh;
            s += dels;
            if (fabs(dels) < fabs(s) * 1e-17) break;
        }
        h = a1 * h;
        kmu = sqrt(CUDART_PI / (2.0 * x)) * exp(-x) / s;
        k1 = kmu * (mu + x + 0.5 - h) / x;
    }
    const double x2i = 2.0 / x;
    for (int i = 1; i <= g.nl; ++i) {                    // K_{mu+i+1} = 2 (mu+i)/x K_{mu+i} + K_{mu+i-1}
        const double kt = (mu + i) * x2i * k1 + kmu;
        kmu = k1;
        k1 = kt;
    }
    const double r = sigma2 * g.pref * exp((mu + g.nl) * log(x)) * kmu;
    // K_nu(x) ~ Gamma(nu)/2 (2/x)^nu overflows for a large nu at a tiny x, where C = sigma2 (1 - O(x^2))
    return isfinite(r) ? r : sigma2;
}

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

template <int NU2>  // 2*nu: 1 -> nu = 1/2, 3 -> nu = 3/2, 5 -> nu = 5/2; sigma2 * C(x) from e = sigma2 exp(-x) (0: general nu)
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
        if (NU2 == 0) {                                   // general nu: Temme / CF2 per element
#pragma unroll
            for (int h = 0; h < RPT; ++h) {
                const double dx = rx[h] - xc, dy = ry[h] - yc;
                v[h] = matern_general(sqrt(fma(dx, dx, dy * dy)) * ib, sigma2, p.gen);
            }
        } else if (fast) {
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

// Host side of the general-nu K1: nu = nl + mu, |mu| <= 1/2 (nl = round(nu)), the Gamma terms of
// Temme's series in long double — gam1 = (1/Gamma(1-mu) - 1/Gamma(1+mu)) / (2 mu) by its Taylor form
// -gamma + (gamma zeta(2)/2 - zeta(3)/3 - gamma^3/6) mu^2 where the difference would cancel (|mu| <
// 1e-4), gam2 = (1/Gamma(1-mu) + 1/Gamma(1+mu)) / 2 — and the iteration reciprocals.
void matern_general_setup(double nu, MaternGen &g) {
    const int nl = (int)floor(nu + 0.5);
    const long double mu = (long double)nu - nl;
    const long double pi = 3.141592653589793238462643383279502884L;
    const long double eg = 0.577215664901532860606512090082402431L, z2 = pi * pi / 6, z3 = 1.202056903159594285399738161511449991L;
    const long double gampl = 1.0L / tgammal(1.0L + mu), gammi = 1.0L / tgammal(1.0L - mu);
    g.mu = (double)mu;
    g.nl = nl;
    g.gp = (double)tgammal(1.0L + mu);
    g.gm = (double)tgammal(1.0L - mu);
    g.gam2 = (double)(0.5L * (gammi + gampl));
    g.gam1 = fabsl(mu) < 1e-4L ? (double)(-eg + (eg * z2 / 2 - z3 / 3 - eg * eg * eg / 6) * mu * mu)
                               : (double)((gammi - gampl) / (2.0L * mu));
    g.fact = fabsl(mu) < 1e-12L ? 1.0 : (double)(pi * mu / sinl(pi * mu));
    g.pref = (double)(powl(2.0L, 1.0L - (long double)nu) / tgammal((long double)nu));
    for (int k = 0; k < matg::TMAX; ++k) {
        g.rq[k] = k ? (double)(1.0L / ((long double)k * k - mu * mu)) : 0.0;
        g.rim[k] = k ? (double)(1.0L / ((long double)k - mu)) : 0.0;
        g.rip[k] = k ? (double)(1.0L / ((long double)k + mu)) : 0.0;
    }
    const long double a1 = 0.25L - mu * mu;
    for (int i = 0; i < matg::CMAX; ++i) {
        const long double ai = -a1 - (long double)i * (i - 1);
        g.ria[i] = i >= 2 ? (double)(1.0L / ai) : 0.0;
        g.rinv[i] = i >= 1 ? (double)(1.0L / i) : 0.0;
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
    else if (nu == 2.5) k1_launch<5>(grid, a, st);
    else {
        matern_general_setup(nu, a.gen);
        k_cov_matern<0, 4, 2><<<grid, 256, 0, st>>>(a);
    }
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
