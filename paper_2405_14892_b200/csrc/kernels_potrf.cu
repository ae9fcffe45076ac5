// K2-K4 — right-looking tiled Cholesky Sigma = L L^T (Alg. 1 line 8; box (a) of P:319).
//
// Per super-panel of kp tile columns (128x128 tiles, lower tile-packed storage):
//   K2 k_potrf_diag2 : A_kk = L_kk L_kk^T in shared memory (one CTA, blocked, DMMA), pivot check -> info
//   K3 k_trsm2       : L_ik = A_ik L_kk^{-T}, i > k (two CTAs per tile, blocked, DMMA)
//   K4 k_update2 / k_update : A_ij -= sum_c L_ic L_jc^T over the super-panel (persistent DMMA GEMM /
//                      two 64x128 CTAs per tile for small counts)
// The paper's StarPU task DAG becomes stream order; the K4 GEMM carries
// n^3/3 of the n^3/3 + O(n^2 nb) flops.
#include <algorithm>
#include <cstdlib>

#include <mutex>

#include "common.cuh"
#include "gemm_dmma.cuh"
#include "mvn_internal.h"

namespace mvn {

// ------------------------------------------------------------------------------------------ K2/K3
// Blocked versions (32-column blocks) of the diagonal POTRF and the panel TRSM. Shared-memory
// matrices are column-major with a padded column stride (== 4 mod 16 doubles) so that the DMMA
// fragment loads are conflict-free. Per 32-column block: a DMMA GEMM applies the already
// finished columns (K = 32 cb), then a short 32-column substitution finishes the block.
namespace blk {
constexpr int SP = kTile + 4;    // 132: diagonal tile / L_kk in smem
constexpr int SPX = 64 + 4;      // 68: a 64-row half of a panel tile
}

// X[m0.., c0..c0+32) -= X[m0.., 0..K) * B(K x 32), B(k, n) = Bm[k * ldb + b0 + n]; rows [r0, r1)
// of the output in 16-row x 16-column warp tiles (DMMA.8x8x4, 2 x 2 blocks per warp).
__device__ __forceinline__ void blk_gemm_sub(double *X, int ldx, int r0, int r1, int c0, int K, const double *Bm, int ldb,
                                             int b0, int warp, int nwarp, int lane) {
    const int mt = (r1 - r0) / 16;
    for (int t = warp; t < mt * 2; t += nwarp) {
        const int m0 = r0 + (t >> 1) * 16, n0 = (t & 1) * 16;
        double acc[2][2][2] = {};
        for (int k = 0; k < K; k += 4) {
            const int kr = k + (lane & 3);
            double fa[2], fb[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) fa[i] = X[kr * ldx + m0 + i * 8 + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 2; ++j) fb[j] = Bm[kr * ldb + b0 + n0 + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int m = m0 + i * 8 + (lane >> 2), n = c0 + n0 + j * 8 + 2 * (lane & 3);
                X[n * ldx + m] -= acc[i][j][0];
                X[(n + 1) * ldx + m] -= acc[i][j][1];
            }
    }
}

// Rows r of X (columns c0..c0+32) solve x L_cc^T = x: x_j = (x_j - sum_{t<j} x_t L(j,t)) / L(j,j),
// L(j,t) = Lm[(lc + t) * ldl + lc + j] (warp-uniform broadcast). One thread per row, the row in 32
// registers, right-looking: once x_j is final it is subtracted from every later x_q at once, so
// the 31 updates of a step are independent; the division by L(j,j) is a product with rd[j] =
// 1 / L(j,j) (shared memory, from the factorisation), so the critical path is 32 multiplies, not
// 32 divisions or the 528 dependent FMAs of the dot-product order. Fully unrolled (static register
// indices); a rolled step loop with registers rotating down one place per step has a 20x smaller
// code but executes 2x the instructions and measured 2-5x slower (k_potrf_diag2 100 us, k_trsm2
// 78 us against 60 / 17 us).
__device__ __forceinline__ void blk_solve32(double *X, int ldx, int c0, int r, const double *Lm, int ldl, int lc,
                                            const double *rd) {
    double x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = X[(c0 + j) * ldx + r];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const double *Lj = Lm + (lc + j) * ldl + lc;      // column j of the block: L(q, j) = Lj[q]
        x[j] *= rd[j];
#pragma unroll
        for (int q = 1; q < 32; ++q)                      // constant trip count: fully unrolled
            if (q > j) x[q] -= x[j] * Lj[q];
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) X[(c0 + j) * ldx + r] = x[j];
}

// One warp factors the 32 x 32 diagonal block at (c0, c0) of A (column-major, ld): lane i holds row
// i in registers; step j broadcasts the pivot and column j by shuffles (right-looking, the same
// operations in the same order as a column-by-column shared-memory factorisation, except that the
// column is scaled by rsqrt(d_jj), computed beside sqrt(d_jj) instead of a division after it: the
// step's critical path is shuffle, rsqrt, multiply, shuffle, FMA). rd[j] = rsqrt(d_jj) for the
// substitution below the block. Returns the first non-positive pivot's column in the block (-1:
// all positive); the block is written back only when it succeeded.
__device__ __forceinline__ int blk_potrf32(double *A, int ld, int c0, int lane, double *rd) {
    double d[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) d[q] = q <= lane ? A[(c0 + q) * ld + c0 + lane] : 0.0;
    int bad = -1;                                        // (no early exit: keeps the loop unrolled)
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const double djj = __shfl_sync(0xffffffffu, d[j], j);
        if (bad < 0 && !(djj > 0.0)) bad = j;              // warp-uniform
        const double ljj = sqrt(djj), rinv = rsqrt(djj);
        const double lij = lane > j ? d[j] * rinv : lane == j ? ljj : d[j];
        d[j] = lij;
        if (lane == 0) rd[j] = rinv;
#pragma unroll
        for (int q = 1; q < 32; ++q)                      // constant trip count: fully unrolled
            if (q > j) {
                const double lqj = __shfl_sync(0xffffffffu, lij, q);
                if (lane >= q) d[q] -= lij * lqj;
            }
    }
    if (bad >= 0) return bad;
#pragma unroll
    for (int q = 0; q < 32; ++q)
        if (q <= lane) A[(c0 + q) * ld + c0 + lane] = d[q];
    return -1;
}

// The 32-column block loops of K2 / K3: rolled (MVN_PANEL_CB_ROLLED=1, one copy of the block code)
// or unrolled by the compiler (default: 4 copies)
#if defined(MVN_PANEL_CB_ROLLED) && MVN_PANEL_CB_ROLLED
#define MVN_CB_UNROLL _Pragma("unroll 1")
#else
#define MVN_CB_UNROLL
#endif

// K2 (blocked): POTRF of the 128 x 128 diagonal tile k in shared memory. Per 32-column block cb:
// DMMA update of rows >= 32cb by the finished columns, one-warp factorisation of the 32 x 32
// diagonal block (first non-positive pivot -> *info, global row), substitution of the rows below.
__global__ void __launch_bounds__(256) k_potrf_diag2(const TileMap tm, int k, int64_t *__restrict__ info) {
    using namespace blk;
    extern __shared__ double A[];          // [128 cols][SP]
    __shared__ double rdg[kTile];          // 1 / L(j, j)
    __shared__ int failed;
    double *T = tm.tile(k, k);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < kTile * kTile / 2; e += 256) {
        const int col = e >> 6, seg = e & 63;
        cp_async16(A + col * SP + seg * 2, T + col * kTile + seg * 2);
    }
    cp_async_commit();
    if (tid == 0) failed = (*info >= 0);
    cp_async_wait<0>();
    __syncthreads();
    if (failed) return;
    MVN_CB_UNROLL
    for (int cb = 0; cb < 4; ++cb) {
        const int c0 = cb * 32;
        if (cb > 0) {
            blk_gemm_sub(A, SP, c0, kTile, c0, c0, A, SP, c0, warp, 8, lane);
            __syncthreads();
        }
        if (warp == 0) {                   // 32 x 32 diagonal block, lane = row
            const int bad = blk_potrf32(A, SP, c0, lane, rdg + c0);
            if (bad >= 0 && lane == 0) { failed = 1; *info = (int64_t)k * kTile + c0 + bad; }
        }
        __syncthreads();
        if (failed) return;
        const int r = c0 + 32 + tid;
        if (r < kTile) blk_solve32(A, SP, c0, r, A, SP, c0, rdg + c0);
        __syncthreads();
    }
    for (int e = tid; e < kTile * kTile; e += 256) {
        const int col = e >> 7, row = e & 127;
        T[e] = (row >= col) ? A[col * SP + row] : 0.0;
    }
}

// K3 (blocked): L_ik = A_ik L_kk^{-T} for one 64-row half of panel tile i (grid: 2 CTAs per tile).
// The tiles are the selected rows i > k (rs: all rows, or a process row's row blocks from rs.lo on);
// L_kk is read through `dg` (the same storage, or the 2-D factorisation's panel buffer).
__global__ void __launch_bounds__(256) k_trsm2(const TileMap tm, const TileMap dg, int k, const RowSel rs) {
    using namespace blk;
    extern __shared__ double sh[];
    double *X = sh;                        // [128 cols][SPX]: rows h*64 .. h*64+63 of A_ik
    double *Lk = sh + kTile * SPX;         // [128 cols][SP]
    __shared__ double rdk[kTile];          // 1 / L_kk(j, j)
    const int64_t lo = rs.lo > k + 1 ? rs.lo : k + 1;
    const int i = (int)rs.nth_raw(rs.raw(lo) + (blockIdx.x >> 1)), h = blockIdx.x & 1;
    double *Ti = tm.tile(i, k) + h * 64;
    const double *Lkk = dg.tile(k, k);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < kTile * 32; e += 256) {           // 128 cols x 32 pieces
        const int col = e >> 5, seg = e & 31;
        cp_async16(X + col * SPX + seg * 2, Ti + col * kTile + seg * 2);
    }
    for (int e = tid; e < kTile * 64; e += 256) {           // 128 cols x 64 pieces
        const int col = e >> 6, seg = e & 63;
        cp_async16(Lk + col * SP + seg * 2, Lkk + col * kTile + seg * 2);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (tid < kTile) rdk[tid] = 1.0 / Lk[tid * SP + tid];
    __syncthreads();
    MVN_CB_UNROLL
    for (int cb = 0; cb < 4; ++cb) {
        const int c0 = cb * 32;
        if (cb > 0) {
            blk_gemm_sub(X, SPX, 0, 64, c0, c0, Lk, SP, c0, warp, 8, lane);
            __syncthreads();
        }
        if (tid < 64) blk_solve32(X, SPX, c0, tid, Lk, SP, c0, rdk + c0);
        __syncthreads();
    }
    for (int e = tid; e < kTile * 32; e += 256) {
        const int col = e >> 5, seg = e & 31;
        *reinterpret_cast<double2 *>(Ti + col * kTile + seg * 2) = *reinterpret_cast<const double2 *>(X + col * SPX + seg * 2);
    }
}

// ------------------------------------------------------------------------------------------ K4
namespace upd {
constexpr int BM = 64, BN = 128, BK = 16, STAGES = 3;
constexpr int SA = BM + 4, SB = BN + 4;  // == 4 (mod 16)
constexpr int WM = 4, WN = 8;
constexpr int SMEM = STAGES * BK * (SA + SB) * 8;
}  // namespace upd

// Trailing update, one CTA per (tile (i,j), row half h): C(64x128) -= L_ik[h-half] * L_jk^T.
// 4 warps as 2 (M) x 2 (N), warp tile 32x64 = 4x8 DMMA blocks (64 fp64 accumulators / thread).
// dst: where C lives; src: where the panel's tiles L_ik, L_jk are read (the same storage, or the
// broadcast panel buffer of the distributed factorisation).
template <bool MAPPED>   // as k_update2
__global__ void __launch_bounds__(128, 2) k_update(const TileMap dst, const TileMap src, const TileMap srcB, int k, int kp,
                                                   int nt, int c0, int cs, int cb, const RowSel rs) {
    using namespace upd;
    extern __shared__ double sm[];
    double *As = sm;
    double *Bs = sm + STAGES * BK * SA;
    const int64_t id = blockIdx.x >> 1;
    const int h = blockIdx.x & 1;
    // id -> tile (ti, tj) of the column-major enumeration over the selected tile columns (> k+kp-1);
    // the panel is the kp tile columns k .. k+kp-1 (K = 128 kp; tiles (ti, k..k+kp-1) are contiguous).
    int ti, tj, col = 0;
    int64_t base = 0;
    if (MAPPED) upd_item_sel(id, nt, c0, cs, cb, rs, ti, tj, base, col);
    else upd_item(id, nt, c0, cs, cb, ti, tj, base, col);
    const double *__restrict__ Lik = (MAPPED ? src.tile(ti, k) : src.base + tile_offset(ti, k)) + h * BM;   // column stride 128
    const double *__restrict__ Ljk = MAPPED ? srcB.tile(tj, k) : src.base + tile_offset(tj, k);
    double *C = (MAPPED ? dst.tile(ti, tj) : dst.base + tile_offset(ti, tj)) + h * BM;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * 64;
    double acc[WM][WN][2];
#pragma unroll
    for (int a = 0; a < WM; ++a)
#pragma unroll
        for (int b = 0; b < WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    auto load = [&](int ch, int st) {
        const int kc = ch * BK;
        double *as = As + st * BK * SA;
        double *bs = Bs + st * BK * SB;
        // A: 16 columns x 64 rows -> 512 x 16B; 4 per thread
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = q * 128 + tid;       // 0..511
            const int col = e >> 5, seg = e & 31;
            cp_async16(as + col * SA + seg * 2, Lik + (int64_t)(kc + col) * kTile + seg * 2);
        }
        // B: 16 columns x 128 rows -> 1024 x 16B; 8 per thread
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = q * 128 + tid;
            const int col = e >> 6, seg = e & 63;
            cp_async16(bs + col * SB + seg * 2, Ljk + (int64_t)(kc + col) * kTile + seg * 2);
        }
    };
    gemm_mainloop<BK, STAGES, SA, SB, WM, WN>(kp * (kTile / BK), As, Bs, wm0, wn0, lane, acc, load);

    // epilogue: C[row][col] -= acc, C column-major (column stride 128); loads batched per row block
#pragma unroll
    for (int a = 0; a < WM; ++a) {
        const int row = wm0 + a * 8 + (lane >> 2);
        double cv[WN][2];
#pragma unroll
        for (int b = 0; b < WN; ++b) {
            const double *p0 = C + (int64_t)(wn0 + b * 8 + 2 * (lane & 3)) * kTile + row;
            cv[b][0] = p0[0];
            cv[b][1] = p0[kTile];
        }
#pragma unroll
        for (int b = 0; b < WN; ++b) {
            double *p0 = C + (int64_t)(wn0 + b * 8 + 2 * (lane & 3)) * kTile + row;
            p0[0] = cv[b][0] - acc[a][b][0];
            p0[kTile] = cv[b][1] - acc[a][b][1];
        }
    }
}

// ------------------------------------------------------------------------------------------ K4
// Persistent trailing update (the hot loop of the Cholesky): CTA c processes tiles
// c, c + grid, ... of the trailing lower triangle (column by column). Per tile C_ij -= L_ik L_jk^T
// (128 x 128 x 128):
//   warp 8 (producer): per 8-column K-chunk, the 8 columns of L_ik and L_jk (cp.async, completion
//                     tracked on the stage's mbarrier) into a 4-stage ring (full/empty mbarriers);
//   warps 0-7        : warp w owns 16 full columns of the tile (warp tile 128 x 16 = 16 x 2
//                      DMMA.8x8x4 blocks, 64 fp64 accumulators / thread). Epilogue: -acc is
//                      written to the warp's 16 KB staging buffer in the tile's column-major
//                      layout and ONE TMA bulk reduction (cp.reduce.async.bulk .add.f64) adds it
//                      to C in L2 — no global loads, nothing to wait for before the next tile.
// The producer runs ahead across tiles, so the next tile's operands stream in during the epilogue.
// K-columns per ring stage and stages of k_update2 (same bytes in flight, BK * STAGES = 32);
// compile-time MVN_UPD2_BK for experiments: 16 x 2 measured 1.1 % slower than 8 x 4 at D and E
// (round-1 A/B, profiles/r01_sov_evolution.md), unlike the SOV ring where fewer, larger chunks won
#ifndef MVN_UPD2_BK
#define MVN_UPD2_BK 8
#endif
namespace upd2 {
constexpr int BK = MVN_UPD2_BK, STAGES = 32 / MVN_UPD2_BK;
constexpr int SP = kTile + 4;                       // 132 == 4 (mod 16)
constexpr int STAGE = 2 * BK * SP;                  // A and B chunks
constexpr int NCONS = 256, NT = NCONS + 32;
constexpr int OFF_STG = STAGES * STAGE;             // [8 warps][16 cols][128 rows]
constexpr int OFF_BAR = OFF_STG + 8 * 16 * kTile;
constexpr int SMEM = (OFF_BAR + 2 * STAGES) * 8;
constexpr int CHUNKS = kTile / BK;
}  // namespace upd2

__device__ __forceinline__ void bulk_reduce_add_f64(double *gdst, const double *ssrc, unsigned bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n"
                 ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// Updates with panel k the tile columns c0, c0 + cs, ... (c0 > k): c0 = k+2, cs = 1 on one GPU
// (column k+1 is the lookahead stream's); cs = world size for the 1-D block-cyclic distributed
// factorisation (mvn_potrf_update).
// MAPPED = false: the full lower tile-packed buffer (dst.base == src.base, tile_offset addressing —
// mvn_potrf's hot loop, register-lean); true: explicit TileMaps (NEXT-1 distributed storage).
template <bool MAPPED>
__global__ void __launch_bounds__(upd2::NT, 1) k_update2(const TileMap dst, const TileMap src, const TileMap srcB, int k,
                                                        int kp, int nt, int c0, int cs, int cb, int64_t nitems,
                                                        const RowSel rs) {
    using namespace upd2;
    extern __shared__ double sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
    uint64_t *empty = full + STAGES;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCONS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    int64_t base = 0;
    int col = 0;
    uint32_t q = 0;
    if (tid >= NCONS) {
        // ------------------------------------------------------------ producer warp
        const int lane = tid & 31;
        for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
            int ti, tj;
            if (MAPPED) upd_item_sel(item, nt, c0, cs, cb, rs, ti, tj, base, col);
            else upd_item(item, nt, c0, cs, cb, ti, tj, base, col);
            // kp consecutive tiles (a super-panel row is contiguous in every TileMap)
            const double *Lik = MAPPED ? src.tile(ti, k) : src.base + tile_offset(ti, k);
            const double *Ljk = MAPPED ? srcB.tile(tj, k) : src.base + tile_offset(tj, k);
            for (int c = 0; c < kp * CHUNKS; ++c, ++q) {
                const int st = q % STAGES;
                mbar_wait(&empty[st], ((q / STAGES) & 1) ^ 1);
                double *as = sm + st * STAGE;
                double *bs = as + BK * SP;
                // BK columns of L_ik and of L_jk (1 KB each) into padded rows: cp.async, 16 B per lane
                const double *a0 = Lik + (int64_t)c * BK * kTile + lane * 2;
                const double *b0 = Ljk + (int64_t)c * BK * kTile + lane * 2;
#pragma unroll
                for (int t = 0; t < BK; ++t)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {                // 1 KB column = 2 x 32 lanes x 16 B
                        cp_async16(as + t * SP + h * 64 + lane * 2, a0 + (int64_t)t * kTile + h * 64);
                        cp_async16(bs + t * SP + h * 64 + lane * 2, b0 + (int64_t)t * kTile + h * 64);
                    }
                cp_async_mbar_arrive(&full[st]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[st]);
            }
        }
        return;
    }
    // ---------------------------------------------------------------- consumer warps
    const int lane = tid & 31, warp = tid >> 5;
    const int wn0 = warp * 16;                       // 16 full columns per warp
    double *stg = sm + OFF_STG + warp * 16 * kTile;   // column-major [16][128]
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        int ti, tj;
        if (MAPPED) upd_item_sel(item, nt, c0, cs, cb, rs, ti, tj, base, col);
        else upd_item(item, nt, c0, cs, cb, ti, tj, base, col);
        double acc[16][2][2];
#pragma unroll
        for (int a = 0; a < 16; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        for (int c = 0; c < kp * CHUNKS; ++c, ++q) {
            const int st = q % STAGES;
            mbar_wait(&full[st], (q / STAGES) & 1);
            const double *as = sm + st * STAGE;
            const double *bs = as + BK * SP;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double fa[16], fb[2];
                const int kr = kk + (lane & 3);
#pragma unroll
                for (int b = 0; b < 2; ++b) fb[b] = bs[kr * SP + wn0 + b * 8 + (lane >> 2)];
#pragma unroll
                for (int a = 0; a < 16; ++a) fa[a] = as[kr * SP + a * 8 + (lane >> 2)];
#pragma unroll
                for (int a = 0; a < 16; ++a)
#pragma unroll
                    for (int b = 0; b < 2; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        // epilogue: the previous tile's reduction must have finished reading the staging buffer
        if (lane == 0) bulk_wait_read_all();
        __syncwarp();
#pragma unroll
        for (int a = 0; a < 16; ++a) {
            const int row = a * 8 + (lane >> 2);
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int cl = b * 8 + 2 * (lane & 3);
                stg[cl * kTile + row] = -acc[a][b][0];
                stg[(cl + 1) * kTile + row] = -acc[a][b][1];
            }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes -> async proxy
        __syncwarp();
        if (lane == 0)
            bulk_reduce_add_f64((MAPPED ? dst.tile(ti, tj) : dst.base + tile_offset(ti, tj)) + (int64_t)wn0 * kTile, stg,
                                16 * kTile * 8);
    }
    if (lane == 0) bulk_wait_all();
}

cudaError_t potrf_init() {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_update<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, upd::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_update<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, upd::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_update2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, upd2::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_update2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, upd2::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_potrf_diag2, cudaFuncAttributeMaxDynamicSharedMemorySize, kTile * blk::SP * 8))) return e;
    if ((e = cudaFuncSetAttribute(k_trsm2, cudaFuncAttributeMaxDynamicSharedMemorySize, kTile * (blk::SP + blk::SPX) * 8))) return e;
    return cudaSuccess;
}

// Streams and events of the single-GPU lookahead schedule (launch_potrf).
namespace {
// SMs left to the panel stream beside the persistent update (MVN_POTRF_PANEL_SMS overrides).
// Measured at D (r01, kp = 4): 4 / 6 / 8 / 12 SMs -> 2.814 / 2.825 / 2.845 / 2.925 s; with kp = 8
// (round-1 A/B): 2 / 4 / 6 / 8 SMs -> 2.805 / 2.786 / 2.778 / 2.792 s (4 kept: within 0.3 %).
int panel_sms() {
    static const int v = [] { const char *e = getenv("MVN_POTRF_PANEL_SMS"); const int x = e ? atoi(e) : 4; return x >= 0 && x < 64 ? x : 4; }();
    return v;
}
// One panel stream and its events per device (created on first use, kept for the process; a
// process may drive several devices). The per-device mutex makes the enqueue of one factorisation
// atomic with respect to other host threads using the same device: the events are re-recorded by
// every call, and a stream-wait captures the latest record at enqueue time.
struct PotrfStreams {
    bool ready = false;
    cudaStream_t sp = nullptr;
    cudaEvent_t ev_panel[2] = {}, ev_rest[2] = {}, ev_start = nullptr;
    std::mutex mu;
};
constexpr int kMaxDevices = 64;
PotrfStreams g_ps_dev[kMaxDevices];
// caller holds ps.mu
cudaError_t potrf_streams(PotrfStreams &ps) {
    if (ps.ready) return cudaSuccess;
    int lo = 0, hi = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (e != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithPriority(&ps.sp, cudaStreamNonBlocking, hi))) return e;
    for (int i = 0; i < 2; ++i) {
        if ((e = cudaEventCreateWithFlags(&ps.ev_panel[i], cudaEventDisableTiming))) return e;
        if ((e = cudaEventCreateWithFlags(&ps.ev_rest[i], cudaEventDisableTiming))) return e;
    }
    if ((e = cudaEventCreateWithFlags(&ps.ev_start, cudaEventDisableTiming))) return e;
    ps.ready = true;
    return cudaSuccess;
}
}  // namespace

// ---- building blocks shared by mvn_potrf and the distributed factorisation (identical arithmetic)
// Factor the kp tile columns k .. k+kp-1 (all updates from columns < k applied): POTRF + TRSM of
// column k; for each further column k+j: update it with columns k .. k+j-1 (K = 128 j), POTRF, TRSM.
// row_end < nt: only the rows < row_end (the 2-D factorisation's diagonal block).
cudaError_t launch_potrf_panel_map(int64_t n, const TileMap &tm, int k, int kp, int64_t *d_info, cudaStream_t st,
                                   int row_end) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int ne = (row_end <= 0 || row_end > nt) ? nt : row_end;
    kp = std::min(kp, nt - k);
    const size_t sm_diag = kTile * blk::SP * 8, sm_trsm = kTile * (blk::SP + blk::SPX) * 8;
    const RowSel all;
    for (int j = 0; j < kp; ++j) {
        const int c = k + j;
        if (j > 0) {
            if (tm.mode == TileMap::kFull && ne == nt)
                k_update<false><<<(unsigned)(2 * (nt - c)), 128, upd::SMEM, st>>>(tm, tm, tm, k, j, nt, c, nt, 1, all);
            else k_update<true><<<(unsigned)(2 * (ne - c)), 128, upd::SMEM, st>>>(tm, tm, tm, k, j, ne, c, ne, 1, all);
        }
        k_potrf_diag2<<<1, 256, sm_diag, st>>>(tm, c, d_info);
        if (ne - c - 1 > 0) k_trsm2<<<2 * (ne - c - 1), 256, sm_trsm, st>>>(tm, tm, c, all);
    }
    return cudaGetLastError();
}

// 2-D factorisation, the process column of super-panel (k, w): the selected (owned) rows >= k + w of
// the local storage `tm` solved against the factored diagonal block read from the panel buffer `pb`:
// per column c = k + j: update by the columns k .. c-1 (L_i from tm, L_c from pb), then TRSM with L_cc.
cudaError_t launch_panel_trsm_map(int64_t n, const TileMap &tm, const TileMap &pb, int k, int w, const RowSel &rs,
                                  cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    w = std::min(w, nt - k);
    RowSel sel = rs;
    sel.lo = k + w;
    const int64_t rows = sel.count(nt);
    if (rows <= 0) return cudaSuccess;
    const size_t sm_trsm = kTile * (blk::SP + blk::SPX) * 8;
    for (int j = 0; j < w; ++j) {
        const int c = k + j;
        if (j > 0) k_update<true><<<(unsigned)(2 * rows), 128, upd::SMEM, st>>>(tm, tm, pb, k, j, nt, c, nt, 1, sel);
        k_trsm2<<<(unsigned)(2 * rows), 256, sm_trsm, st>>>(tm, pb, c, sel);
    }
    return cudaGetLastError();
}
cudaError_t launch_potrf_panel(int64_t n, double *tiles, int k, int kp, int64_t *d_info, cudaStream_t st) {
    return launch_potrf_panel_map(n, TileMap::full(tiles), k, kp, d_info, st, 0);
}

// A_ij -= sum_{c=k}^{k+kp-1} L_ic L_jc^T for the tile columns j = c0 + m cs + b (0 <= b < cb) and
// i >= j: the persistent kernel (on nsm - sm_reserve SMs) when there are >= 2 tiles per CTA, else
// two CTAs per tile.
cudaError_t launch_potrf_update_map(int64_t n, const TileMap &dst, const TileMap &src, int k, int kp, int c0, int cs,
                                    int cb, int sm_reserve, cudaStream_t st) {
    return launch_potrf_update_map(n, dst, src, src, k, kp, c0, cs, cb, sm_reserve, RowSel(), st);
}

// dst: the updated storage; srcA / srcB: where L_ik / L_jk are read; rs: the rows of dst updated.
cudaError_t launch_potrf_update_map(int64_t n, const TileMap &dst, const TileMap &src, const TileMap &srcB, int k, int kp,
                                    int c0, int cs, int cb, int sm_reserve, const RowSel &rs, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    if (c0 >= nt) return cudaSuccess;
    kp = std::min(kp, nt - k);
    const bool sel = rs.P != 1 || rs.lo > 0;
    const int64_t items = sel ? upd_items_sel(nt, c0, cs, cb, rs) : upd_items(nt, c0, cs, cb);
    if (items == 0) return cudaSuccess;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    static const bool use_persistent = [] { const char *e = getenv("MVN_POTRF_PERSISTENT"); return !(e && e[0] == '0'); }();
    const int avail = std::max(1, nsm - sm_reserve);
    const bool mapped = dst.mode != TileMap::kFull || src.mode != TileMap::kFull || dst.base != src.base ||
                        srcB.mode != TileMap::kFull || srcB.base != src.base || sel;
    if (use_persistent && items >= 2 * avail) {
        if (mapped) k_update2<true><<<avail, upd2::NT, upd2::SMEM, st>>>(dst, src, srcB, k, kp, nt, c0, cs, cb, items, rs);
        else k_update2<false><<<avail, upd2::NT, upd2::SMEM, st>>>(dst, src, srcB, k, kp, nt, c0, cs, cb, items, rs);
    } else {
        if (mapped) k_update<true><<<(unsigned)(2 * items), 128, upd::SMEM, st>>>(dst, src, srcB, k, kp, nt, c0, cs, cb, rs);
        else k_update<false><<<(unsigned)(2 * items), 128, upd::SMEM, st>>>(dst, src, srcB, k, kp, nt, c0, cs, cb, rs);
    }
    return cudaGetLastError();
}
cudaError_t launch_potrf_update(int64_t n, double *tiles, int k, int kp, int c0, int cs, int cb, int sm_reserve,
                                cudaStream_t st) {
    const TileMap tm = TileMap::full(tiles);
    return launch_potrf_update_map(n, tm, tm, k, kp, c0, cs, cb, sm_reserve, st);
}

// Super-panel width for an order-n factorisation: wider panels cut the update passes (K = 128 kp
// per pass) but lengthen the panel chain on the critical path. Measured on B200 (r01, CUDA events):
//   n = 16,384  kp 1 / 2 / 3      = 60 / 64 / 66 ms
//   n = 32,761  kp 1 / 2 / 3      = 409 / 390 / 384 ms
//   n = 65,536  kp 1 / 2 / 3 / 4  = 3.14 / 2.96 / 2.89 / 2.86 s
//   n = 102,400 kp 2 / 3 / 4      = 11.21 / 10.96 / 10.83 s
// and with the final kernels (r01 A/B on one box):
//   n = 25,600  kp 3 / 6 / 8      = 199 / 201 / 203 ms
//   n = 65,536  kp 4 / 6 / 8      = 2.822 / 2.805 / 2.791 s
//   n = 102,400 kp 4 / 6 / 8      = 10.57 / 10.46 / 10.39 s
// MVN_POTRF_KP (1..8) overrides.
int potrf_panel_sms() { return panel_sms(); }

int potrf_panel_width(int64_t n) {
    static const int env = [] { const char *e = getenv("MVN_POTRF_KP"); const int v = e ? atoi(e) : 0; return v >= 1 && v <= 8 ? v : 0; }();
    if (env) return env;
    const int64_t nt = (n + kTile - 1) / kTile;
    return nt >= 384 ? 8 : nt >= 192 ? 3 : 1;
}

// Right-looking factorisation over super-panels of kp = potrf_panel_width() tile columns (K = 128 kp
// per trailing update: half the update passes and epilogues of a 128-wide step), with one step of
// lookahead on two streams:
//   panel stream (high priority): update of the next super-panel's columns with super-panel s, then
//                                 its factorisation (launch_potrf_panel);
//   main stream                 : persistent update of the columns after the next super-panel, on
//                                 all but panel_sms() SMs, so the panel work runs beside it.
// Events order the two (panel s before update s; update s-1 before the panel-stream update of s).
cudaError_t launch_potrf(int64_t n, double *tiles, int64_t *d_info, cudaStream_t st, int ncols) {
    return launch_potrf_ex(n, tiles, d_info, st, ncols, nullptr);
}

// oz != nullptr: the main-stream trailing updates on the int8 tensor cores (NEXT-4 mixed precision,
// kernels_potrf_oz.cu); the panel stream (look-ahead update + panel factorisation) stays fp64. An
// int8 update pays only with wide super-panels (K = 128 kp: the per-tile TMEM drain and the per-step
// slicing are fixed costs) and enough tiles to fill the clusters: below kp = 8 (n < 49,152) or
// 4 tiles per cluster the update runs on fp64 DMMA (measured at C, kp = 1: 184 ms int8 vs 60 ms).
// MVN_POTRF_OZ_ALWAYS=1 (read per call; tests) takes the int8 path for every trailing update.
static bool use_oz(const PotrfOz *oz, int nt, int kp, int c0) {
    if (!oz) return false;
    const char *e = getenv("MVN_POTRF_OZ_ALWAYS");
    if (e && e[0] == '1') return true;
    return kp >= 8 && upd_items(nt, c0, 1, 1) >= 4ll * oz->clusters;
}

cudaError_t launch_potrf_ex(int64_t n, double *tiles, int64_t *d_info, cudaStream_t st, int ncols, const PotrfOz *oz) {
    const int nt = (int)((n + kTile - 1) / kTile);
    if (ncols <= 0 || ncols > nt) ncols = nt;      // ncols < nt: partial factorisation (Schur complement left)
    const int KP = potrf_panel_width(n);
    const int S = (ncols + KP - 1) / KP;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    PotrfStreams &ps = g_ps_dev[dev];
    std::lock_guard<std::mutex> lock(ps.mu);
    cudaError_t e = potrf_streams(ps);
    if (e != cudaSuccess) return e;
    cudaStream_t sp = ps.sp;
    // the panel stream starts after everything already queued on the main stream (Sigma)
    if ((e = cudaEventRecord(ps.ev_start, st))) return e;
    if ((e = cudaStreamWaitEvent(sp, ps.ev_start, 0))) return e;
    if ((e = launch_potrf_panel(n, tiles, 0, std::min(KP, ncols), d_info, sp))) return e;
    if ((e = cudaEventRecord(ps.ev_panel[0], sp))) return e;
    for (int s = 0; s < S; ++s) {
        const int k = s * KP, w = std::min(KP, ncols - k);
        const int kn = k + w;
        if ((e = cudaStreamWaitEvent(st, ps.ev_panel[s & 1], 0))) return e;
        if (s + 1 == S) {
            // last super-panel: the trailing (Schur complement) block of a partial factorisation
            if (kn < nt) {
                e = use_oz(oz, nt, KP, kn) ? launch_potrf_update_oz(n, tiles, k, w, kn, 1, 1, oz->clusters, oz->LAp, oz->rs, oz->xch, st)
                       : launch_potrf_update(n, tiles, k, w, kn, 1, 1, 0, st);
                if (e) return e;
            }
            break;
        }
        const int wn = std::min(KP, ncols - kn);
        // main stream: columns >= kn + wn with super-panel s
        e = use_oz(oz, nt, KP, kn + wn) ? launch_potrf_update_oz(n, tiles, k, w, kn + wn, 1, 1, oz->clusters_reserved, oz->LAp, oz->rs, oz->xch, st)
               : launch_potrf_update(n, tiles, k, w, kn + wn, 1, 1, panel_sms(), st);
        if (e) return e;
        if ((e = cudaEventRecord(ps.ev_rest[s & 1], st))) return e;
        // panel stream: columns kn .. kn+wn-1 with super-panel s, then factor super-panel s+1
        if (s >= 1 && (e = cudaStreamWaitEvent(sp, ps.ev_rest[(s - 1) & 1], 0))) return e;
        if ((e = launch_potrf_update(n, tiles, k, w, kn, nt, wn, 0, sp))) return e;
        if ((e = launch_potrf_panel(n, tiles, kn, wn, d_info, sp))) return e;
        if ((e = cudaEventRecord(ps.ev_panel[(s + 1) & 1], sp))) return e;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------ NEXT-1
// Building blocks of the distributed (1-D block-cyclic over super-panels of kp tile columns)
// factorisation; the step loop and the NCCL panel broadcasts live in
// paper_2405_14892_b200/parallel.py (collectives stay above the ABI). Every rank keeps a full
// tile-packed buffer; it updates only the tile columns it owns and receives every other super-panel
// finished, so each rank ends with all of L. launch_potrf_panel / launch_potrf_update above are the
// arithmetic; this adds the panel copy.

// Super-panel copy between two storages: the tiles (i, c), k <= c < k + kp, i >= c, from one
// TileMap to another (full storage or a rank's owned columns <-> the kPanel broadcast buffer, whose
// tiles run row after row so that a super-panel row (i, k .. k+kp-1) is contiguous).
// grid (8, tiles of the super-panel): one CTA per (tile, 1/8).
__global__ void __launch_bounds__(256) k_panel_copy(const TileMap from, const TileMap to, int k, int nt) {
    int idx = blockIdx.y, c = k;
    while (idx >= nt - c) { idx -= nt - c; ++c; }
    const int i = c + idx;
    if (!from.owns_row(i) || !to.owns_row(i)) return;     // 2-D storage: another process row's tile
    const double2 *f = reinterpret_cast<const double2 *>(from.tile(i, c));
    double2 *t = reinterpret_cast<double2 *>(to.tile(i, c));
    constexpr int PER = kTile * kTile / 2 / 8;             // double2 per CTA
    const int e0 = blockIdx.x * PER;
#pragma unroll 4
    for (int e = threadIdx.x; e < PER; e += 256) t[e0 + e] = f[e0 + e];
}

cudaError_t launch_panel_copy_map(int64_t n, const TileMap &from, const TileMap &to, int k, int kp, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    kp = std::min(kp, nt - k);
    int ntiles = 0;
    for (int j = 0; j < kp; ++j) ntiles += nt - k - j;
    if (ntiles == 0) return cudaSuccess;
    k_panel_copy<<<dim3(8, ntiles), 256, 0, st>>>(from, to, k, nt);
    return cudaGetLastError();
}

// Tile-row copy: the tiles (i, j), tb <= i < te, j <= i, that `from` owns, to their places in `to`
// (the row slice of mvn_sweep_rows: a full map whose base is offset to tile row tb). grid (8, tiles
// of the rows, 8): one CTA per (tile, 1/8), row-major tile enumeration from (tb, 0).
__global__ void __launch_bounds__(256) k_rows_copy(const TileMap from, const TileMap to, int tb) {
    const int64_t id = (int64_t)blockIdx.x + (int64_t)tb * (tb + 1) / 2;
    int ti = (int)((sqrt(8.0 * (double)id + 1.0) - 1.0) * 0.5);
    while ((int64_t)ti * (ti + 1) / 2 > id) --ti;
    while ((int64_t)(ti + 1) * (ti + 2) / 2 <= id) ++ti;
    const int tj = (int)(id - (int64_t)ti * (ti + 1) / 2);
    if (!from.owns_col(tj) || !from.owns_row(ti)) return;
    const double2 *f = reinterpret_cast<const double2 *>(from.tile(ti, tj));
    double2 *t = reinterpret_cast<double2 *>(to.tile(ti, tj));
    constexpr int PER = kTile * kTile / 2 / 8;
    const int e0 = blockIdx.y * PER;
#pragma unroll 4
    for (int e = threadIdx.x; e < PER; e += 256) t[e0 + e] = f[e0 + e];
}

cudaError_t launch_rows_copy_map(const TileMap &from, const TileMap &to, int tb, int te, cudaStream_t st) {
    const int64_t ntiles = (int64_t)te * (te + 1) / 2 - (int64_t)tb * (tb + 1) / 2;
    if (ntiles <= 0) return cudaSuccess;
    k_rows_copy<<<dim3((unsigned)ntiles, 8), 256, 0, st>>>(from, to, tb);
    return cudaGetLastError();
}

cudaError_t launch_panel_copy(int64_t n, double *tiles, int k, int kp, double *panel, bool to_panel, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const TileMap full = TileMap::full(tiles), pan = TileMap::panel(panel, k, std::min(kp, nt - k));
    return to_panel ? launch_panel_copy_map(n, full, pan, k, kp, st) : launch_panel_copy_map(n, pan, full, k, kp, st);
}

}  // namespace mvn
