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
#include "common.cuh"
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
__device__ __forceinline__ int rr_col(int pos, int s) { return pos == 0 ? 0 : 1 + (pos - 1 + s) % (tlr::NB - 1); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(tlr::NT, 1) k_tlr_compress(double *__restrict__ tiles, int nt, double eps, int mode,
                                                            int *__restrict__ ranks) {
    using namespace tlr;
    extern __shared__ double sh[];
    double *X = sh;                               // [128 cols][LD]: A, then R, then R^T rotated
    double *wb = X + NB * LD;                     // [NW warps][2][128]
    double *vb = wb + 2 * NW * NB;                // Householder vector
    double *cn = vb + NB;                         // squared norms of the trailing sub-columns
    int *perm = reinterpret_cast<int *>(cn + NB); // column pivots: (A P)(:, r) = A(:, perm[r])
    __shared__ int chgf[2], k_sel, piv;
    __shared__ double vtv_s, fro2_s;
    __shared__ double sig[NB], srt[NB];
    __shared__ int sel[NB], pos[NB];
    (void)nt;
    // off-diagonal tile index -> (I, J), I > J
    const int64_t t = blockIdx.x;
    int I = (int)((sqrt(8.0 * (double)t + 1.0) + 1.0) * 0.5);
    while ((int64_t)I * (I - 1) / 2 > t) --I;
    while ((int64_t)(I + 1) * I / 2 <= t) ++I;
    const int J = (int)(t - (int64_t)I * (I - 1) / 2);
    double *T = tiles + tile_offset(I, J);
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

    // ---- 1. column-pivoted Householder QR (R overwrites A; the reflectors are not kept)
    for (int j = 0; j < NB; ++j) {
        if (warp == 0) {                          // pivot: largest trailing norm, lowest index on ties
            double bv = -1.0;
            int bi = j;
#pragma unroll
            for (int m = 0; m < NB / 32; ++m) {
                const int c = lane + 32 * m;
                if (c >= j && cn[c] > bv) { bv = cn[c]; bi = c; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
            }
            if (lane == 0) piv = bi;
        }
        __syncthreads();
        const int p = piv;
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
    for (int sweep = 0; sweep < MAX_SWEEPS; ++sweep) {
        // flag slot of this sweep; the other slot is the one a lagging warp may still be reading for
        // the previous sweep's exit test
        int &chg = chgf[sweep & 1];
        if (tid == 0) chg = 0;
        __syncthreads();
        for (int s = 0; s < NB - 1; ++s) {
            const int p = warp + NW * grp;
            double *ai = X + rr_col(p, s) * LD, *aj = X + rr_col(NB - 1 - p, s) * LD;
            double2 x[NB / 16], y[NB / 16];       // elements 2 l8 + 16 m (+1)
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
            if (fabs(ga) > 1e-15 * sqrt(al * be) && ga != 0.0 && al + be >= floor2) {
                const double zeta = (be - al) / (2.0 * ga);
                const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + tt * tt), sn = c * tt;
#pragma unroll
                for (int m = 0; m < NB / 16; ++m) {
                    *reinterpret_cast<double2 *>(ai + 2 * l8 + 16 * m) = make_double2(c * x[m].x - sn * y[m].x, c * x[m].y - sn * y[m].y);
                    *reinterpret_cast<double2 *>(aj + 2 * l8 + 16 * m) = make_double2(sn * x[m].x + c * y[m].x, sn * x[m].y + c * y[m].y);
                }
                if (l8 == 0) chg = 1;
            }
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
        }
        __syncwarp();
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
    k_tlr_compress<<<(unsigned)noff, tlr::NT, tlr::SMEM, st>>>(tiles, nt, eps, mode, ranks);
    return cudaGetLastError();
}

}  // namespace mvn
