// Device primitives shared by the libmvn kernels (sm_100a only).
//  - fp64 tensor-core MMA: mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4. tcgen05 has no f64 kind on
//    sm_100a (ptxas rejects .kind::f64), so warp-level DMMA with register operands is the fp64
//    tensor path; measured 37.07 TFLOP/s = the chip's fp64 peak (profiles/r01_fp64_calibration.md).
//  - cp.async 16-byte global->shared copies (LDGSTS) for multi-stage operand pipelines.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "mvn_internal.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libmvn is built for sm_100a (B200) only"
#endif

namespace mvn {

__host__ __device__ inline int64_t tile_offset(int64_t i, int64_t j) {
    return ((i * (i + 1)) / 2 + j) * (int64_t)kTile * kTile;
}

// Where tile (i, j), i >= j, of a lower tile-packed matrix lives (128 x 128 column-major tiles):
//   kFull : every lower tile, row after row — tile_offset(i, j);
//   kDist : only the tile columns a rank owns under the 1-D block-cyclic map of super-panels of kp
//           columns over W ranks (super-panel s = columns s kp .. s kp + kp - 1, owned by rank
//           s mod W), row after row: (owned tiles in rows < i) + (owned columns < j). A rank's
//           memory is ~1/W of the matrix (NEXT-1 distributed storage);
//   kPanel: the tiles (i, k .. min(i, k + kp - 1)), i >= k, of the super-panel (k, kp), row after
//           row (the broadcast buffer of the distributed factorisation).
// In every mode the tiles (i, c .. c + m) of one super-panel row are consecutive in memory.
//   2-D  : kDist with P > 1 process rows — the tile rows are distributed too (row block I = i / kp
//           owned by process row I mod P): a rank (pr, g) holds the tiles (i, j) of its row blocks
//           and column blocks, row after row (2-D block-cyclic over a P x W grid, NEXT-1).
struct TileMap {
    enum : int { kFull = 0, kDist = 1, kPanel = 2 };
    double *base = nullptr;
    int mode = kFull, W = 1, g = 0, kp = 1, k = 0;
    int P = 1, pr = 0;                                     // process rows (kDist 2-D)

    // owned columns in [0, x) (kDist)
    __host__ __device__ int64_t owned_below(int64_t x) const {
        const int64_t P = (int64_t)kp * W, r = x % P - (int64_t)g * kp;
        return (x / P) * kp + (r < 0 ? 0 : r > kp ? kp : r);
    }
    // owned tiles in tile rows < i = sum_{x=1..i} owned_below(x) (kDist), closed form
    __host__ __device__ int64_t owned_rows_below(int64_t i) const {
        const int64_t P = (int64_t)kp * W, T = i + 1, Q = T / P, R = T % P, K = kp;
        const int64_t H = K * (K - 1) / 2 + K * (P - (int64_t)(g + 1) * K);
        const int64_t u = R - (int64_t)g * K;
        const int64_t Hp = u <= 0 ? 0 : u <= K ? u * (u - 1) / 2 : K * (K - 1) / 2 + K * (u - K);
        return P * K * Q * (Q - 1) / 2 + Q * H + R * Q * K + Hp;
    }
    // owned tiles in the tile rows < i of this rank's row blocks (kDist, 2-D): per owned row block B
    // the rows x give owned_below(x + 1) tiles each, i.e. owned_rows_below((B+1) kp) - owned_rows_below(B kp)
    __host__ __device__ int64_t owned_rows_below_2d(int64_t i) const {
        const int64_t I = i / kp;
        int64_t t = 0;
        for (int64_t B = pr; B < I; B += P) t += owned_rows_below((B + 1) * kp) - owned_rows_below(B * kp);
        if (I % P == pr) t += owned_rows_below(i) - owned_rows_below(I * kp);
        return t;
    }
    __host__ __device__ int64_t index(int64_t i, int64_t j) const {
        if (mode == kFull) return (i * (i + 1)) / 2 + j;
        if (mode == kDist) return (P == 1 ? owned_rows_below(i) : owned_rows_below_2d(i)) + owned_below(j);
        const int64_t m = i - k;
        return (m <= kp ? m * (m + 1) / 2 : (int64_t)kp * (kp + 1) / 2 + (m - kp) * kp) + (j - k);
    }
    __host__ __device__ double *tile(int64_t i, int64_t j) const { return base + index(i, j) * (int64_t)kTile * kTile; }
    __host__ __device__ bool owns_col(int64_t j) const { return mode != kDist || (j / kp) % W == g; }
    __host__ __device__ bool owns_row(int64_t i) const { return mode != kDist || P == 1 || (i / kp) % P == pr; }
    static TileMap full(double *b) { TileMap m; m.base = b; return m; }
    static TileMap dist(double *b, int W_, int g_, int kp_) { TileMap m; m.base = b; m.mode = kDist; m.W = W_; m.g = g_; m.kp = kp_; return m; }
    static TileMap panel(double *b, int k_, int kp_) { TileMap m; m.base = b; m.mode = kPanel; m.k = k_; m.kp = kp_; return m; }
    static TileMap dist2(double *b, int P_, int pr_, int Q_, int pc_, int kp_) {
        TileMap m = dist(b, Q_, pc_, kp_);
        m.P = P_; m.pr = pr_;
        return m;
    }
};

// Row selection of the update enumerations: the tile rows i >= lo whose row block i / kp is owned by
// process row pr of P (P = 1, lo = 0: every row).
struct RowSel {
    int P = 1, pr = 0, kp = 1, lo = 0;
    // selected rows in [0, x)
    __host__ __device__ int64_t count(int64_t x) const {
        if (x <= lo) return 0;
        return raw(x) - raw(lo);
    }
    __host__ __device__ int64_t raw(int64_t x) const {
        if (P == 1) return x;
        const int64_t Pk = (int64_t)kp * P, r = x % Pk - (int64_t)pr * kp;
        return (x / Pk) * kp + (r < 0 ? 0 : r > kp ? kp : r);
    }
    // the row of raw index idx (the idx-th owned row counted from row 0)
    __host__ __device__ int64_t nth_raw(int64_t idx) const {
        if (P == 1) return idx;
        return (idx / kp) * (int64_t)kp * P + (int64_t)pr * kp + idx % kp;
    }
};

// Column-major enumeration of the trailing tiles (ti, tj), ti >= tj, over the tile columns
//   tj = c0 + m*cs + b,  m >= 0, 0 <= b < cb,  tj < nt
// (blocks of cb consecutive columns every cs columns; cb = cs = 1: every column from c0; the
// distributed factorisation passes cb = kp, cs = kp * W). Column tj holds nt - tj tiles. `base` /
// `col` carry the scan between calls (the items of one CTA increase monotonically).
__host__ __device__ inline int upd_col(int idx, int c0, int cs, int cb) { return c0 + (idx / cb) * cs + idx % cb; }

__device__ __forceinline__ void upd_item(int64_t item, int nt, int c0, int cs, int cb, int &ti, int &tj, int64_t &base,
                                         int &col) {
    while (item >= base + (nt - upd_col(col, c0, cs, cb))) { base += nt - upd_col(col, c0, cs, cb); ++col; }
    tj = upd_col(col, c0, cs, cb);
    ti = tj + (int)(item - base);
}

__host__ __device__ inline int64_t upd_items(int nt, int c0, int cs, int cb) {
    int64_t s = 0;
    for (int idx = 0; upd_col(idx, c0, cs, cb) < nt; ++idx) s += nt - upd_col(idx, c0, cs, cb);
    return s;
}

// The same with a row selection: column tj holds the selected rows i >= tj.
__host__ __device__ inline int64_t upd_col_count(const RowSel &rs, int nt, int tj) {
    const int64_t lo = rs.lo > tj ? rs.lo : tj;
    return lo >= nt ? 0 : rs.raw(nt) - rs.raw(lo);
}
__device__ __forceinline__ void upd_item_sel(int64_t item, int nt, int c0, int cs, int cb, const RowSel &rs, int &ti,
                                             int &tj, int64_t &base, int &col) {
    while (item >= base + upd_col_count(rs, nt, upd_col(col, c0, cs, cb))) {
        base += upd_col_count(rs, nt, upd_col(col, c0, cs, cb));
        ++col;
    }
    tj = upd_col(col, c0, cs, cb);
    const int64_t lo = rs.lo > tj ? rs.lo : tj;
    ti = (int)rs.nth_raw(rs.raw(lo) + (item - base));
}
__host__ __device__ inline int64_t upd_items_sel(int nt, int c0, int cs, int cb, const RowSel &rs) {
    int64_t s = 0;
    for (int idx = 0; upd_col(idx, c0, cs, cb) < nt; ++idx) s += upd_col_count(rs, nt, upd_col(idx, c0, cs, cb));
    return s;
}

// C(8x8) += A(8x4, row) * B(4x8, col). Fragment ownership (lane l):
//   a = A[l/4][l%4], b = B[l%4][l/4], c = {C[l/4][2(l%4)], C[l/4][2(l%4)+1]}
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- named barriers, mbarriers and TMA bulk copies (SASS: BAR, SYNCS.*, UBLKCP)
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// TMA-engine bulk copy global -> shared, completion counted on an mbarrier (SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Arrive on an mbarrier when all of this thread's prior cp.async copies have landed (the pending
// count is raised now and dropped at completion, so the phase cannot complete before them).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Bulk prefetch of a global range into L2 (no shared-memory destination).
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace mvn
