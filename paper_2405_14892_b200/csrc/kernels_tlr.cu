// NEXT-3 (part) — Tile Low-Rank compression of the covariance at a fixed accuracy (§II-C,
// "the separate approximation of each tile using the Singular Value Decomposition ...
// the ranks of the tiles correspond to the most significant singular values"; Alg. 1 l.7, P:248:
// pmvn_init "encompasses the compression of the covariance matrix Sigma into the TLR format").
// Reading R23: an off-diagonal 128 x 128 tile keeps its k largest singular triplets,
// k set by the accuracy eps: mode 0, sigma_i >= eps (absolute, on a unit-variance Sigma); mode 1,
// the smallest k with ||A - A_k||_F <= eps ||A||_F (relative per tile). Diagonal tiles stay dense.
//
// One CTA per off-diagonal tile, the tile (column-major) in shared memory:
//  1. column-pivoted Householder QR, A P = Q R (Q is not kept);
//  2. X = R^T, orthogonalised by one-sided Jacobi (Hestenes) rotations in round-robin column pairs
//     until every pair is orthogonal to 1e-15 relative (pairs of columns both below 1e-3 eps
//     excepted). The QR preconditioning (Drmac-Veselic) cuts the sweeps from 24-37 to 8-12 on the
//     Matérn tiles and is what makes the iteration converge within its sweep cap there
//     (tools/tlr_jacobi_sweeps.py). X's columns are then u_i sigma_i with R^T = U_x Sigma W^T, so
//     the right singular vectors of A are v_i = P u_i;
//  3. k from eps (mode above); each row of A (re-read from global memory) is projected onto
//     span(v_1..v_k): A~ = A V_k V_k^T = U_k Sigma_k V_k^T, written back in place (the compressed
//     tile in reconstructed form, which the dense POTRF / SOV consume unchanged); k is recorded.
// Work is O(sweeps * 128^3) per tile on the fp64 ALU; used for the accuracy study, not on the
// timed path.
#include <vector>

#include "common.cuh"
#include "gemm_dmma.cuh"
#include "mvn_internal.h"

namespace mvn {
namespace tlr {
// LD even (16-byte aligned columns): the Jacobi steps move columns as double2, an 8-lane group
// covering 128 contiguous bytes per access, so a warp request is exactly 4 wavefronts whatever the
// 4 columns are; strided phases (transpose, phase 3) use a skewed index order instead
constexpr int NB = kTile, LD = kTile + 2, NT = 512, NW = NT / 32, MAX_SWEEPS = 30;
constexpr int SMEM = (NB * LD + 2 * NW * NB + 2 * NB) * 8 + NB * 4;
}  // namespace tlr

// column at position `pos` of step s of a round-robin (circle-method) pairing of 128 columns:
// position 0 fixed, positions 1..127 rotate; pair p = (pos p, pos 127 - p).
// (m even: the first m columns; positions 0 .. m-1)
__device__ __forceinline__ int rr_col(int pos, int s, int m) { return pos == 0 ? 0 : 1 + (pos - 1 + s) % (m - 1); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Where the tiles come from and where the result goes (TlrJob):
//  src_mode 0: every off-diagonal tile (I, J) of the full tile-packed buffer, t = blockIdx.x;
//  src_mode 1: the tiles (i, j), i = j + 1 + blockIdx.x, of one tile column held in the panel
//              workspace (tile i at src + (i - j) 128^2; the TLR Cholesky, R26), t = i(i-1)/2 + j;
//  src_mode 2: the same tiles of column j read from the full tile-packed buffer;
//  U == nullptr: the compressed tile is written back in place (reconstructed, R23);
//  U != nullptr: the factors are written instead, U_t = A V_k (128 x k) and V_t = V_k (128 x k),
//              column-major in the slot t of stride 128 kmax; a rank above kmax sets *overflow and
//              is stored as kmax (the caller reports MVN_E_NOMEM).
struct TlrJob {
    double *src = nullptr;
    int src_mode = 0, j = 0;
    double *U = nullptr, *V = nullptr;
    int kmax = 0;
    int *overflow = nullptr;
};

// 1/x, sqrt(x), 1/sqrt(x) for normal positive (rcp: nonzero) x: the MUFU fp64 seed (~2^-23) and
// Newton steps (quadratic: two reach ~2^-46, the third ~1 ulp)
__device__ __forceinline__ double rcp_nr(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
    for (int i = 0; i < 3; ++i) y = y * fma(-0.5 * x, y * y, 1.5);
    return y;
}
__device__ __forceinline__ double sqrt_nr(double x) {
    const double y = rsqrt_nr(x), t = x * y;
    return fma(fma(-t, t, x), 0.5 * y, t);          // one Newton correction of t = x / sqrt(x)
}

__global__ void __launch_bounds__(tlr::NT, 1) k_tlr_compress(const TlrJob job, double eps, int mode,
                                                            int *__restrict__ ranks) {
    using namespace tlr;
    extern __shared__ double sh[];
    double *X = sh;                               // [128 cols][LD]: A, then R, then R^T rotated
    double *wb = X + NB * LD;                     // [NW warps][2][128]
    double *vb = wb + 2 * NW * NB;                // Householder vector
    double *cn = vb + NB;                         // squared norms of the trailing sub-columns
    int *perm = reinterpret_cast<int *>(cn + NB); // column pivots: (A P)(:, r) = A(:, perm[r])
    __shared__ int chgf[2], k_sel, piv, kq_s;
    __shared__ double vtv_s, fro2_s;
    __shared__ double sig[NB], srt[NB];
    __shared__ int sel[NB], pos[NB];
    int64_t t;
    double *T;
    if (job.src_mode == 0) {              // off-diagonal tile index -> (I, J), I > J
        t = blockIdx.x;
        int I = (int)((sqrt(8.0 * (double)t + 1.0) + 1.0) * 0.5);
        while ((int64_t)I * (I - 1) / 2 > t) --I;
        while ((int64_t)(I + 1) * I / 2 <= t) ++I;
        const int J = (int)(t - (int64_t)I * (I - 1) / 2);
        T = job.src + tile_offset(I, J);
    } else {
        const int64_t i = (int64_t)job.j + 1 + blockIdx.x;
        t = i * (i - 1) / 2 + job.j;
        T = job.src_mode == 1 ? job.src + (i - job.j) * (int64_t)NB * NB : job.src + tile_offset(i, job.j);
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < NB * NB; e += NT) X[(e >> 7) * LD + (e & 127)] = T[e];
    if (tid < NB) perm[tid] = tid;
    __syncthreads();
    for (int c = warp; c < NB; c += NW) {
        double s2 = 0.0;
#pragma unroll
        for (int m = 0; m < NB / 32; ++m) s2 = fma(X[c * LD + lane + 32 * m], X[c * LD + lane + 32 * m], s2);
        s2 = warp_sum(s2);
        if (lane == 0) cn[c] = s2;
    }
    __syncthreads();
    if (warp == 0) {                              // ||A||_F^2 (the scale of the mode-1 Jacobi floor)
        double f = 0.0;
#pragma unroll
        for (int m = 0; m < NB / 32; ++m) f += cn[lane + 32 * m];
        f = warp_sum(f);
        if (lane == 0) fro2_s = f;
    }

    // ---- 1. column-pivoted Householder QR (R overwrites A; the reflectors are not kept). It stops at
    // step kq once the trailing block's Frobenius norm ||R_22||_F (the sum of the trailing column norms
    // cn) is <= tau = 1e-6 of the truncation scale: R_22 is dropped, which moves every singular value
    // by <= ||R_22||_2 <= tau, and the Jacobi below then works on kq columns instead of 128 (the
    // low-rank tiles of a TLR matrix stop early)
    const double tau2 = 1e-12 * eps * eps * (mode == 1 ? fro2_s : 1.0);
    if (tid == 0) kq_s = NB;
    for (int j = 0; j < NB; ++j) {
        if (warp == 0) {                          // pivot: largest trailing norm, lowest index on ties
            double bv = -1.0, tot = 0.0;
            int bi = j;
#pragma unroll
            for (int m = 0; m < NB / 32; ++m) {
                const int c = lane + 32 * m;
                if (c >= j) {
                    tot += cn[c];
                    if (cn[c] > bv) { bv = cn[c]; bi = c; }
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
            }
            tot = warp_sum(tot);
            if (lane == 0) piv = tot <= tau2 ? -1 : bi;
        }
        __syncthreads();
        const int p = piv;
        if (p < 0) {                              // ||R_22||_F <= tau: R = [R_11 R_12; 0 0]
            for (int e = tid; e < (NB - j) * NB; e += NT) {
                const int c = j + e / NB, r = e % NB;
                if (r >= j) X[c * LD + r] = 0.0;
            }
            if (tid == 0) kq_s = j;
            __syncthreads();
            break;
        }
        if (p != j) {
            if (tid < NB) {
                const double a = X[j * LD + tid];
                X[j * LD + tid] = X[p * LD + tid];
                X[p * LD + tid] = a;
            }
            if (tid == NB) {
                const int q = perm[j];
                perm[j] = perm[p];
                perm[p] = q;
                cn[p] = cn[j];
            }
            __syncthreads();
        }
        if (warp == 0) {                          // reflector H = I - 2 v v^T / (v^T v) mapping x to alpha e_j
            double x[NB / 32], s2 = 0.0;
#pragma unroll
            for (int m = 0; m < NB / 32; ++m) {
                const int r = lane + 32 * m;
                x[m] = r >= j ? X[j * LD + r] : 0.0;
                s2 = fma(x[m], x[m], s2);
            }
            s2 = warp_sum(s2);
            const double x0 = X[j * LD + j], xn = sqrt(s2);
            const double alpha = -copysign(xn, x0), v0 = x0 - alpha;
#pragma unroll
            for (int m = 0; m < NB / 32; ++m) {
                const int r = lane + 32 * m;
                if (r >= j) {
                    vb[r] = (r == j) ? v0 : x[m];
                    X[j * LD + r] = (r == j) ? (xn > 0.0 ? alpha : x0) : 0.0;
                }
            }
            if (lane == 0) vtv_s = xn > 0.0 ? s2 - x0 * x0 + v0 * v0 : 0.0;
        }
        __syncthreads();
        const double vtv = vtv_s;
        for (int c = j + 1 + warp; c < NB; c += NW) {
            double d = 0.0;
            double y[NB / 32];
#pragma unroll
            for (int m = 0; m < NB / 32; ++m) {
                const int r = lane + 32 * m;
                y[m] = r >= j ? X[c * LD + r] : 0.0;
                if (r >= j) d = fma(vb[r], y[m], d);
            }
            d = warp_sum(d);
            const double f = vtv > 0.0 ? 2.0 * d / vtv : 0.0;
            double s2 = 0.0;
#pragma unroll
            for (int m = 0; m < NB / 32; ++m) {
                const int r = lane + 32 * m;
                if (r >= j) {
                    y[m] = fma(-f, vb[r], y[m]);
                    X[c * LD + r] = y[m];
                    if (r > j) s2 = fma(y[m], y[m], s2);
                }
            }
            s2 = warp_sum(s2);
            if (lane == 0) cn[c] = s2;
        }
        __syncthreads();
    }
    // X = R^T (lower triangular)
    for (int e = tid; e < NB * NB; e += NT) {
        const int c = e & 127, i = ((e >> 7) + c) & 127;   // skewed: lanes hit distinct banks
        if (i > c) {
            X[c * LD + i] = X[i * LD + c];
            X[i * LD + c] = 0.0;
        }
    }
    __syncthreads();

    // ---- 2. one-sided Jacobi on X: an 8-lane group per column pair, 4 pairs per warp, 64 per step
    const int grp = lane >> 3, l8 = lane & 7;
    const unsigned gmask = 0xffu << (grp * 8);
    // pairs whose two columns together are below 1e-3 of the truncation scale stay unrotated: 1e-3 eps
    // (mode 0, absolute sigma_i >= eps) or 1e-3 eps ||A||_F (mode 1, relative: scale-invariant)
    const double floor2 = 1e-6 * eps * eps * (mode == 1 ? fro2_s : 1.0);
    // the columns of X past kq are zero: rotate only the first kq (rounded up to even; a zero column
    // never rotates)
    const int mq = kq_s + (kq_s & 1);
    // this group's pair: positions p and mq - 1 - p; the columns there at step s are
    // rr_col(pos, s), advanced by one per step (mq - 1 -> 1; position 0 fixed) instead of a runtime
    // modulo per step (two integer divisions, ~60 instructions)
    const int pg = warp + NW * grp;
    int ca = pg, cb = mq - 1 - pg;
    for (int sweep = 0; sweep < MAX_SWEEPS && mq > 1; ++sweep) {
        // flag slot of this sweep; the other slot is the one a lagging warp may still be reading for
        // the previous sweep's exit test
        int &chg = chgf[sweep & 1];
        if (tid == 0) chg = 0;
        __syncthreads();
        for (int s = 0; s < mq - 1; ++s) {
            const bool active = 2 * pg < mq;      // a pair for this 8-lane group (none past mq / 2)
            if (active) {
                double *ai = X + ca * LD, *aj = X + cb * LD;
                double2 x[NB / 16], y[NB / 16];   // elements 2 l8 + 16 m (+1)
                double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
                for (int m = 0; m < NB / 16; ++m) {
                    x[m] = *reinterpret_cast<const double2 *>(ai + 2 * l8 + 16 * m);
                    y[m] = *reinterpret_cast<const double2 *>(aj + 2 * l8 + 16 * m);
                    al = fma(x[m].x, x[m].x, fma(x[m].y, x[m].y, al));
                    be = fma(y[m].x, y[m].x, fma(y[m].y, y[m].y, be));
                    ga = fma(x[m].x, y[m].x, fma(x[m].y, y[m].y, ga));
                }
#pragma unroll
                for (int o = 4; o; o >>= 1) {
                    al += __shfl_xor_sync(gmask, al, o);
                    be += __shfl_xor_sync(gmask, be, o);
                    ga += __shfl_xor_sync(gmask, ga, o);
                }
                if (ga * ga > 1e-30 * al * be && ga != 0.0 && al + be >= floor2) {   // |ga| > 1e-15 sqrt(al be), no sqrt
                    // rotation (c, s) from MUFU-seeded reciprocals / square roots refined by Newton
                    // steps (~1 ulp; the IEEE div / sqrt sequences were the step's longest latency chain)
                    const double zeta = be == al ? 0.0 : (be - al) * rcp_nr(2.0 * ga);   // (no 0 * inf for a subnormal ga)
                    const double az = fabs(zeta);
                    const double tt = az > 1e100 ? 0.5 / zeta                 // 1 / (2 zeta): sqrt(1 + zeta^2) ~ |zeta|
                                                 : copysign(rcp_nr(az + sqrt_nr(fma(zeta, zeta, 1.0))), zeta);
                    const double c = rsqrt_nr(fma(tt, tt, 1.0)), sn = c * tt;
#pragma unroll
                    for (int m = 0; m < NB / 16; ++m) {
                        *reinterpret_cast<double2 *>(ai + 2 * l8 + 16 * m) = make_double2(c * x[m].x - sn * y[m].x, c * x[m].y - sn * y[m].y);
                        *reinterpret_cast<double2 *>(aj + 2 * l8 + 16 * m) = make_double2(sn * x[m].x + c * y[m].x, sn * x[m].y + c * y[m].y);
                    }
                    if (l8 == 0) chg = 1;
                }
            }
            if (ca != 0) ca = ca == mq - 1 ? 1 : ca + 1;
            cb = cb == mq - 1 ? 1 : cb + 1;
            __syncthreads();
        }
        if (!chg) break;
    }

    // ---- 3. singular values, kept set, normalised u_i; rows of A projected onto span(P u_i)
    if (tid < NB) {
        double s2 = 0.0;
        for (int r = 0; r < NB; ++r) s2 = fma(X[tid * LD + r], X[tid * LD + r], s2);
        sig[tid] = sqrt(s2);
    }
    __syncthreads();
    if (tid < NB) {                               // position in descending order (ties: lower index first)
        const double v = sig[tid];
        int p = 0;
#pragma unroll 4
        for (int j = 0; j < NB; ++j) p += (sig[j] > v) || (sig[j] == v && j < tid);
        pos[tid] = p;
        srt[p] = v;
    }
    __syncthreads();
    if (tid == 0) {
        int k = 0;
        if (mode == 0) {                          // absolute: sigma_i >= eps
#pragma unroll 1
            while (k < NB && srt[k] >= eps && srt[k] > 0.0) ++k;
        } else {                                  // relative Frobenius: ||A - A_k||_F <= eps ||A||_F
            double tot = 0.0;
#pragma unroll 1
            for (int i = NB - 1; i >= 0; --i) tot = fma(srt[i], srt[i], tot);
            const double budget = eps * eps * tot;
            double tail = 0.0;
            k = NB;
            while (k > 0 && tail + srt[k - 1] * srt[k - 1] <= budget) {
                tail = fma(srt[k - 1], srt[k - 1], tail);
                --k;
            }
        }
        if (job.U && k > job.kmax) {
            atomicMax(job.overflow, k);
            k = job.kmax;
        }
        k_sel = k;
        ranks[t] = k;
    }
    __syncthreads();
    if (tid < NB && pos[tid] < k_sel) sel[pos[tid]] = tid;
    __syncthreads();
    const int k = k_sel;
    for (int e = tid; e < k * NB; e += NT) {
        const int q = e >> 7, r = e & 127;
        X[sel[q] * LD + r] /= sig[sel[q]];
    }
    __syncthreads();
    double *wa = wb + warp * 2 * NB, *ww = wa + NB;
    double *Ut = nullptr;
    if (job.U) {                                  // factors: V_t(:, q) = P u_sel[q] (the normalised right vectors)
        Ut = job.U + t * (int64_t)NB * job.kmax;
        double *Vt = job.V + t * (int64_t)NB * job.kmax;
        for (int e = tid; e < k * NB; e += NT) {
            const int q = e >> 7, r = e & 127;
            Vt[(int64_t)q * NB + perm[r]] = X[sel[q] * LD + r];
        }
    }
    int pr[NB / 32];
#pragma unroll
    for (int m = 0; m < NB / 32; ++m) pr[m] = perm[lane + 32 * m];
    for (int rho = warp; rho < NB; rho += NW) {
        // a(r) = A(rho, perm[r]); row rho is read and written by this warp only
#pragma unroll
        for (int m = 0; m < NB / 32; ++m) wa[lane + 32 * m] = T[(int64_t)pr[m] * NB + rho];
        __syncwarp();
        for (int q = lane; q < k; q += 32) {      // w_q = u_q^T a
            const double *u = X + sel[q] * LD;
            double d = 0.0;
            for (int r0 = 0; r0 < NB; ++r0) {     // skewed start: the 32 lanes read 32 columns in distinct banks
                const int r = (r0 + q) & (NB - 1);
                d = fma(u[r], wa[r], d);
            }
            ww[q] = d;
            if (Ut) Ut[(int64_t)q * NB + rho] = d;          // U_t(rho, q) = (A V_k)(rho, q)
        }
        __syncwarp();
        if (Ut) continue;
        double out[NB / 32];
#pragma unroll
        for (int m = 0; m < NB / 32; ++m) out[m] = 0.0;
        for (int q = 0; q < k; ++q) {
            const double *u = X + sel[q] * LD;
            const double wq = ww[q];
#pragma unroll
            for (int m = 0; m < NB / 32; ++m) out[m] = fma(u[lane + 32 * m], wq, out[m]);
        }
#pragma unroll
        for (int m = 0; m < NB / 32; ++m) T[(int64_t)pr[m] * NB + rho] = out[m];
        __syncwarp();
    }
}

cudaError_t tlr_init() { return cudaFuncSetAttribute(k_tlr_compress, cudaFuncAttributeMaxDynamicSharedMemorySize, tlr::SMEM); }

cudaError_t launch_tlr_compress(int64_t n, double *tiles, double eps, int mode, int *ranks, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int64_t noff = (int64_t)nt * (nt - 1) / 2;
    if (noff == 0) return cudaSuccess;
    TlrJob job;
    job.src = tiles;
    k_tlr_compress<<<(unsigned)noff, tlr::NT, tlr::SMEM, st>>>(job, eps, mode, ranks);
    return cudaGetLastError();
}


// ============================================================================================
// NEXT-3: the TLR Cholesky (reading R26; oracle/tlr.py tlr_cholesky). Off-diagonal tiles of Sigma
// and of L live as factors U_t V_t^T in slots of 128 x kmax doubles (column-major, t = I(I-1)/2 + J,
// rank r_t); the diagonal tiles are dense in the tile-packed buffer. Tile column j is assembled in a
// dense panel workspace (tile i at pnl + (i - j) 128^2):
//   T_i = Stilde_ij - sum_{k<j} U_ik (V_ik^T V_jk) U_jk^T                        (i >= j)
// as three batched products over (i, k) per chunk of k (M_ik = V_ik^T V_jk, Z_ik = U_ik M_ik,
// T_i -= sum_k Z_ik U_jk^T), then the dense K2 / K3 kernels factor the panel and k_tlr_compress
// truncates each L_ij at eps into its slot. Flops per (i, j, k): 4 128 r_ik r_jk + 2 128^2 r_jk
// (dense: 2 128^3) — the saving is r / 128 when ranks are small.
namespace tlrg {
constexpr int BM = 64, BN = 64, BK = 16, NT = 128, SA = BM + 4, SB = BN + 4;   // SA, SB == 4 (mod 16)
enum : int { kExpandPanel = 0, kExpandAll = 1, kM = 2, kZ = 3, kAcc = 4 };
}  // namespace tlrg

// acc(64 x 64 block at (m0, n0)) += A B over k < K. Every operand has leading dimension 128:
//   A(m, k) = AT ? A[m 128 + k] : A[k 128 + m];   B(k, n) = BKC ? B[n 128 + k] : B[k 128 + n]
// Elements with m >= Md, n >= Nd or k >= K read as 0 (ranks need no padding in the slots).
template <bool AT, bool BKC>
__device__ __forceinline__ void tlr_seg_gemm(double (&c)[4][4][2], const double *__restrict__ A,
                                             const double *__restrict__ B, int K, int Md, int Nd, int m0, int n0,
                                             double *As, double *Bs) {
    using namespace tlrg;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 32;
    const int nch = (K + BK - 1) / BK;
    double ra[8], rb[8];
    auto idx_a = [&](int e, int &kk, int &m) { if (AT) { kk = e & 15; m = e >> 4; } else { kk = e >> 6; m = e & 63; } };
    auto idx_b = [&](int e, int &kk, int &nn) { if (BKC) { kk = e & 15; nn = e >> 4; } else { kk = e >> 6; nn = e & 63; } };
    auto load = [&](int ch) {
        const int k0 = ch * BK;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            int kk, m;
            idx_a(tid + q * NT, kk, m);
            const int gm = m0 + m, gk = k0 + kk;
            ra[q] = (gm < Md && gk < K) ? (AT ? A[(int64_t)gm * 128 + gk] : A[(int64_t)gk * 128 + gm]) : 0.0;
            int kb, nn;
            idx_b(tid + q * NT, kb, nn);
            const int gn = n0 + nn, gkb = k0 + kb;
            rb[q] = (gn < Nd && gkb < K) ? (BKC ? B[(int64_t)gn * 128 + gkb] : B[(int64_t)gkb * 128 + gn]) : 0.0;
        }
    };
    if (nch == 0) return;
    load(0);
    for (int ch = 0; ch < nch; ++ch) {
        __syncthreads();                           // the previous chunk's MMAs are done with As / Bs
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            int kk, m;
            idx_a(tid + q * NT, kk, m);
            As[kk * SA + m] = ra[q];
            int kb, nn;
            idx_b(tid + q * NT, kb, nn);
            Bs[kb * SB + nn] = rb[q];
        }
        __syncthreads();
        if (ch + 1 < nch) load(ch + 1);            // next chunk's global loads in flight under the MMAs
        mma_chunk<BK, SA, SB, 4, 4>(As, Bs, wm0, wn0, lane, c);
    }
}

__device__ __forceinline__ void tlr_cp16(void *smem, const void *gmem, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes));
}

// acc(64 x 64 block at (m0, n0)) += A B over k < K for operands contiguous along the staged rows,
// A(m, k) = A[k 128 + m], B(k, n) = B[k 128 + n] (the expansions U V^T and the accumulation Z U^T):
// a 2-stage cp.async double buffer (rows k >= K zero-filled), one barrier per chunk
__device__ __forceinline__ void tlr_seg_gemm_async(double (&c)[4][4][2], const double *__restrict__ A,
                                                   const double *__restrict__ B, int K, int m0, int n0, double *As2,
                                                   double *Bs2) {
    using namespace tlrg;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 32;
    const int nch = (K + BK - 1) / BK;
    if (nch == 0) return;
    auto issue = [&](int ch, int st) {
        const int k0 = ch * BK;
        double *as = As2 + st * BK * SA, *bs = Bs2 + st * BK * SB;
#pragma unroll
        for (int q = 0; q < 4; ++q) {                     // 16 rows x 32 pieces of 16 bytes, each operand
            const int e = tid + q * NT, kk = e >> 5, pc = e & 31;
            const bool in = k0 + kk < K;
            tlr_cp16(as + kk * SA + 2 * pc, in ? A + (int64_t)(k0 + kk) * 128 + m0 + 2 * pc : A, in ? 16 : 0);
            tlr_cp16(bs + kk * SB + 2 * pc, in ? B + (int64_t)(k0 + kk) * 128 + n0 + 2 * pc : B, in ? 16 : 0);
        }
        cp_async_commit();
    };
    __syncthreads();                                      // the previous segment's readers are done
    issue(0, 0);
    for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait<0>();
        __syncthreads();                                  // chunk ch landed; chunk ch - 1's readers are done
        if (ch + 1 < nch) issue(ch + 1, (ch + 1) & 1);
        mma_chunk<BK, SA, SB, 4, 4>(As2 + (ch & 1) * BK * SA, Bs2 + (ch & 1) * BK * SB, wm0, wn0, lane, c);
    }
}

struct TlrGemm {
    int mode = 0, nt = 0, j = 0, k0 = 0, kc = 0, kmax = 0, nsplit = 1;
    double *tiles = nullptr, *pnl = nullptr, *U = nullptr, *V = nullptr, *Mw = nullptr, *Zw = nullptr;
    const int *ranks = nullptr;
    const int *ranks_s = nullptr;      // Sigma's ranks (kExpandPanel)
};

// grid: (entries, 4 blocks of 64 x 64); 128 threads (2 x 2 warps of 32 x 32); MODE = g.mode
template <int MODE>
__global__ void __launch_bounds__(tlrg::NT) k_tlr_gemm(const TlrGemm g) {
    using namespace tlrg;
    __shared__ __align__(16) double smb[2 * BK * (SA + SB)];
    double *As = smb, *Bs = smb + BK * SA;              // register-staged path (M, Z)
    double *As2 = smb, *Bs2 = smb + 2 * BK * SA;        // cp.async path (expansions, accumulation)
    const int m0 = (blockIdx.y & 1) * BM, n0 = (blockIdx.y >> 1) * BN;
    const int64_t e = blockIdx.x, S = (int64_t)128 * g.kmax, T2 = (int64_t)128 * 128;
    double c[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) c[a][b][0] = c[a][b][1] = 0.0;
    double *C;
    int Md = 128, Nd = 128;
    bool sub = false;
    if (MODE == kExpandPanel || MODE == kExpandAll) {          // C = U_t V_t^T (dense tile)
        int64_t t;
        if (MODE == kExpandPanel) {
            const int64_t i = g.j + 1 + e;
            t = i * (i - 1) / 2 + g.j;
            C = g.pnl + (i - g.j) * T2;
        } else {
            t = e;
            int I = (int)((sqrt(8.0 * (double)t + 1.0) + 1.0) * 0.5);
            while ((int64_t)I * (I - 1) / 2 > t) --I;
            while ((int64_t)(I + 1) * I / 2 <= t) ++I;
            C = g.tiles + tile_offset(I, t - (int64_t)I * (I - 1) / 2);
        }
        tlr_seg_gemm_async(c, g.U + t * S, g.V + t * S, MODE == kExpandPanel ? g.ranks_s[t] : g.ranks[t], m0, n0, As2,
                           Bs2);
    } else if (MODE == kM || MODE == kZ) {
        const int64_t i = g.j + e / g.kc, k = g.k0 + e % g.kc;
        const int64_t tik = i * (i - 1) / 2 + k, tjk = (int64_t)g.j * (g.j - 1) / 2 + k;
        const int rik = g.ranks[tik], rjk = g.ranks[tjk];
        if (MODE == kM) {                                      // M_ik = V_ik^T V_jk  (r_ik x r_jk)
            Md = rik;
            Nd = rjk;
            if (m0 >= Md || n0 >= Nd) return;
            C = g.Mw + e * T2;
            tlr_seg_gemm<true, true>(c, g.V + tik * S, g.V + tjk * S, 128, Md, Nd, m0, n0, As, Bs);
        } else {                                               // Z_ik = U_ik M_ik  (128 x r_jk)
            Nd = rjk;
            if (n0 >= Nd) return;
            C = g.Zw + e * T2;
            tlr_seg_gemm<false, true>(c, g.U + tik * S, g.Mw + e * T2, rik, 128, Nd, m0, n0, As, Bs);
        }
    } else {                                                   // T_i -= sum_k Z_ik U_jk^T
        // nsplit > 1 (few panel tiles): the k range is split over nsplit CTAs per tile, each writing
        // its partial sum to the (consumed) M workspace; k_tlr_reduce subtracts them in order
        const int64_t ii = e / g.nsplit;
        const int sp = (int)(e % g.nsplit);
        const int kb = (int)((int64_t)g.kc * sp / g.nsplit), ke = (int)((int64_t)g.kc * (sp + 1) / g.nsplit);
        if (g.nsplit > 1) {
            C = g.Mw + e * T2;
        } else {
            C = g.pnl + ii * T2;
            sub = true;
        }
        for (int kk = kb; kk < ke; ++kk) {
            const int64_t tjk = (int64_t)g.j * (g.j - 1) / 2 + g.k0 + kk;
            tlr_seg_gemm_async(c, g.Zw + (ii * g.kc + kk) * T2, g.U + tjk * S, g.ranks[tjk], m0, n0, As2, Bs2);
        }
    }
    // c[a][b][h]: row m0 + wm0 + 8a + lane/4, column n0 + wn0 + 8b + 2(lane%4) + h; C column-major (ld 128)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 32;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = m0 + wm0 + 8 * a + (lane >> 2), nn = n0 + wn0 + 8 * b + 2 * (lane & 3) + h;
                double *p = C + (int64_t)nn * 128 + m;
                *p = sub ? *p - c[a][b][h] : c[a][b][h];
            }
}

// T_i -= sum_{s < nsplit} partial(i, s), the partials summed in order (deterministic)
__global__ void __launch_bounds__(256) k_tlr_reduce(double *__restrict__ pnl, const double *__restrict__ part, int nsplit) {
    const int64_t T2 = (int64_t)128 * 128, ii = blockIdx.y;
    const int64_t x = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const double *p = part + ii * nsplit * T2 + x;
    double acc = 0.0;
    for (int s = 0; s < nsplit; ++s) acc += p[s * T2];
    pnl[ii * T2 + x] -= acc;
}

namespace {
cudaError_t tlr_gemm(const TlrGemm &g, int64_t entries, cudaStream_t st) {
    if (entries <= 0) return cudaSuccess;
    const dim3 grid((unsigned)entries, 4);
    switch (g.mode) {
    case tlrg::kExpandPanel: k_tlr_gemm<tlrg::kExpandPanel><<<grid, tlrg::NT, 0, st>>>(g); break;
    case tlrg::kExpandAll: k_tlr_gemm<tlrg::kExpandAll><<<grid, tlrg::NT, 0, st>>>(g); break;
    case tlrg::kM: k_tlr_gemm<tlrg::kM><<<grid, tlrg::NT, 0, st>>>(g); break;
    case tlrg::kZ: k_tlr_gemm<tlrg::kZ><<<grid, tlrg::NT, 0, st>>>(g); break;
    default: k_tlr_gemm<tlrg::kAcc><<<grid, tlrg::NT, 0, st>>>(g); break;
    }
    return cudaGetLastError();
}
}  // namespace

size_t tlr_slot_doubles(int64_t n, int kmax) {
    const int64_t nt = (n + kTile - 1) / kTile;
    return (size_t)(nt * (nt - 1) / 2) * 128 * (size_t)kmax;
}

// Workspace (doubles): two panels (nt tiles each, alternating columns) + M and Z chunks of
// `chunk_slots` tiles each.
size_t tlr_work_doubles(int64_t n, int64_t chunk_slots) {
    const int64_t nt = (n + kTile - 1) / kTile;
    return (size_t)(2 * nt + 2 * chunk_slots) * kTile * kTile;
}

namespace {
// T_i -= sum_{k in [ka, kb)} U_ik (V_ik^T V_jk) U_jk^T for the panel tiles i = j .. nt-1, in chunks
// of at most chunk_slots / rows columns k (M, Z, accumulate; split-K when the column has few tiles)
cudaError_t tlr_update_range(TlrGemm g, int ka, int kb, int64_t chunk_slots, double *Mw, cudaStream_t st) {
    using namespace tlrg;
    const int rows = g.nt - g.j;
    const int kc_max = (int)std::max<int64_t>(1, std::min<int64_t>(kb - ka, chunk_slots / rows));
    cudaError_t e;
    for (int k0 = ka; k0 < kb; k0 += kc_max) {
        g.k0 = k0;
        g.kc = std::min(kc_max, kb - k0);
        g.nsplit = 1;
        g.mode = kM;
        if ((e = tlr_gemm(g, (int64_t)rows * g.kc, st)) != cudaSuccess) return e;
        g.mode = kZ;
        if ((e = tlr_gemm(g, (int64_t)rows * g.kc, st)) != cudaSuccess) return e;
        // few panel tiles: split the k range so that >= ~2 CTAs per SM accumulate
        g.nsplit = (int)std::min<int64_t>(g.kc, std::max<int64_t>(1, (2 * 148 + 4 * rows - 1) / (4 * rows)));
        g.mode = kAcc;
        if ((e = tlr_gemm(g, (int64_t)rows * g.nsplit, st)) != cudaSuccess) return e;
        if (g.nsplit > 1) {
            k_tlr_reduce<<<dim3(128 * 128 / 256, (unsigned)rows), 256, 0, st>>>(g.pnl, Mw, g.nsplit);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

struct SideStream {      // the compression streams of launch_tlr_potrf and their events
    cudaStream_t s = nullptr, sg = nullptr;
    cudaEvent_t panel_done = nullptr, comp_done = nullptr;
    std::vector<cudaEvent_t> sig_done;   // Sigma's column j compressed
    ~SideStream() {
        if (panel_done) cudaEventDestroy(panel_done);
        if (comp_done) cudaEventDestroy(comp_done);
        for (cudaEvent_t e : sig_done) if (e) cudaEventDestroy(e);
        if (s) cudaStreamDestroy(s);     // released once their queued work completes
        if (sg) cudaStreamDestroy(sg);
    }
};
}  // namespace

// Column j's tile compressions (side stream) overlap the next column's updates by the columns
// k < j (main stream); only the k = j term waits for them. The panel alternates between two
// buffers, so column j + 1 is assembled while column j's tiles are still being read.
cudaError_t launch_tlr_potrf(int64_t n, double *tiles, double eps, int mode, int kmax, double *U, double *V,
                             int *ranks, int *ranks_sigma, double *work, int64_t chunk_slots, int *overflow,
                             int64_t *d_info, cudaStream_t st) {
    using namespace tlrg;
    const int nt = (int)((n + kTile - 1) / kTile);
    const int64_t noff = (int64_t)nt * (nt - 1) / 2, T2 = (int64_t)kTile * kTile;
    double *pnls[2] = {work, work + nt * T2};
    double *Mw = work + 2 * nt * T2, *Zw = Mw + chunk_slots * T2;
    cudaError_t e;
    SideStream side;
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (nt > 1 && !ranks_sigma) return cudaErrorInvalidValue;   // the caller provides Sigma's rank array
    // the compressions are on the critical path (column j's factors feed column j + 1): high priority
    if ((e = cudaStreamCreateWithPriority(&side.s, cudaStreamNonBlocking, prio_hi)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&side.panel_done, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&side.comp_done, cudaEventDisableTiming)) != cudaSuccess) return e;
    // (1) Sigma's off-diagonal tiles compressed at eps into the slots (Alg. 1 l.7, R23), column by
    // column on a low-priority stream that runs ahead of the factorisation and fills the SMs its
    // critical path leaves idle; column j's expansion waits for its event. Sigma's ranks go to
    // ranks_sigma (the slots and `ranks` then receive L~'s)
    if ((e = cudaStreamCreateWithPriority(&side.sg, cudaStreamNonBlocking, prio_lo)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(side.comp_done, st)) != cudaSuccess) return e;   // Sigma's tiles are ready (re-recorded per column below)
    if ((e = cudaStreamWaitEvent(side.sg, side.comp_done, 0)) != cudaSuccess) return e;
    side.sig_done.assign((size_t)std::max(nt - 1, 0), nullptr);
    for (int j = 0; j + 1 < nt; ++j) {
        if ((e = cudaEventCreateWithFlags(&side.sig_done[j], cudaEventDisableTiming)) != cudaSuccess) return e;
        TlrJob job;
        job.src = tiles;
        job.src_mode = 2;
        job.j = j;
        job.U = U;
        job.V = V;
        job.kmax = kmax;
        job.overflow = overflow;
        k_tlr_compress<<<(unsigned)(nt - 1 - j), tlr::NT, tlr::SMEM, side.sg>>>(job, eps, mode, ranks_sigma);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = cudaEventRecord(side.sig_done[j], side.sg)) != cudaSuccess) return e;
    }
    TlrGemm g;
    g.nt = nt;
    g.kmax = kmax;
    g.tiles = tiles;
    g.U = U;
    g.V = V;
    g.Mw = Mw;
    g.Zw = Zw;
    g.ranks = ranks;
    g.ranks_s = ranks_sigma;
    for (int j = 0; j < nt; ++j) {
        const int rows = nt - j;                             // panel tiles i = j .. nt-1
        double *pnl = pnls[j & 1];
        g.j = j;
        g.pnl = pnl;
        // T_j = Sigma_jj (dense), T_i = U_ij V_ij^T of Sigma (i > j)
        if ((e = cudaMemcpyAsync(pnl, tiles + tile_offset(j, j), sizeof(double) * T2, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
            return e;
        if (rows > 1 && (e = cudaStreamWaitEvent(st, side.sig_done[j], 0)) != cudaSuccess) return e;
        g.mode = kExpandPanel;
        if ((e = tlr_gemm(g, rows - 1, st)) != cudaSuccess) return e;
        // T_i -= sum_{k<j} U_ik (V_ik^T V_jk) U_jk^T: the columns k < j - 1 while column j - 1 is
        // being compressed, then k = j - 1 after it
        if (j >= 2 && (e = tlr_update_range(g, 0, j - 1, chunk_slots, Mw, st)) != cudaSuccess) return e;
        if (j >= 1) {
            if ((e = cudaStreamWaitEvent(st, side.comp_done, 0)) != cudaSuccess) return e;
            if ((e = tlr_update_range(g, j - 1, j, chunk_slots, Mw, st)) != cudaSuccess) return e;
        }
        // L_jj = chol(T_j), L_ij = T_i L_jj^{-T}: the dense K2 / K3 kernels on the panel
        if ((e = launch_potrf_panel_map(n, TileMap::panel(pnl, j, 1), j, 1, d_info, st, 0)) != cudaSuccess) return e;
        if ((e = cudaMemcpyAsync(tiles + tile_offset(j, j), pnl, sizeof(double) * T2, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
            return e;
        // Ltilde_ij = truncation of L_ij at eps, into slot (i, j), on the side stream
        if (rows > 1) {
            if ((e = cudaEventRecord(side.panel_done, st)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(side.s, side.panel_done, 0)) != cudaSuccess) return e;
            TlrJob job;
            job.src = pnl;
            job.src_mode = 1;
            job.j = j;
            job.U = U;
            job.V = V;
            job.kmax = kmax;
            job.overflow = overflow;
            k_tlr_compress<<<(unsigned)(rows - 1), tlr::NT, tlr::SMEM, side.s>>>(job, eps, mode, ranks);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
            if ((e = cudaEventRecord(side.comp_done, side.s)) != cudaSuccess) return e;
        }
    }
    // join, then the dense SOV reads Ltilde reconstructed (steps (b)-(d) stay dense)
    if ((e = cudaStreamWaitEvent(st, side.comp_done, 0)) != cudaSuccess) return e;
    g.mode = kExpandAll;
    return tlr_gemm(g, noff, st);
}
}  // namespace mvn
