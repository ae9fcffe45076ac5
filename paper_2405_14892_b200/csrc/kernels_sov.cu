// K5/K6 — the SOV sweep with Richtmyer-lattice QMC (Alg. 2 PMVN; Alg. 3 QMC tile
// kernel; Eq. 2-3), all prefixes in one sweep (reading R1).
//
// B200-first decomposition (not the paper's tile-task DAG):
//   * The parallel axis is the sample ("MC chain"). Persistent CTAs, one per SM; CTA c owns
//     a balanced contiguous range of global samples (NR/148 each), swept as blocks of <= 128
//     samples (the last block of a CTA is narrowed to a multiple of 32, so no CTA idles in a tail
//     wave). Each block sweeps all n rows in row blocks of 64.
//   * Warp specialisation (416 threads):
//       warp 12    (producer): streams 32-column K-chunks of the L row panel (from L2 — all CTAs
//                  sweep the same rows) and 32-row chunks of the Y history (this CTA's HBM scratch)
//                  into a 2-stage shared-memory ring with TMA bulk copies (cp.async.bulk, mbarrier
//                  complete_tx); full/empty mbarriers, no CTA-wide barrier in the main loop.
//       warps 0-7  (GEMM): (a6) S_r = L[rows r, 0:64r] * Y[0:64r, block] on fp64 DMMA. The part
//                  of S_{r+1} that only needs Y[0:64r] is computed WHILE the chain warps run row
//                  block r; only the last 64 columns wait for Y_r.
//       warps 8-11 (chain): (a7) Alg. 3's in-block recursion, one thread per sample: sub-blocks of
//                  8 rows, s += in-block dot, Phi/Phi^{-1} step (normal.cuh), ell += log q, y to
//                  the Y history (coalesced) and folded into the remaining rows of S;
//                  (a8) per-row log-sum-exp over the block's samples (warp shuffles).
//     Hand-off through named barriers: S_FULL (GEMM -> chain), Y_READY (chain -> GEMM).
//   * k_reduce_blocks combines the block partials of every prefix in fixed order (deterministic).
// The lattice point w (reading R8) is generated in registers; the n x NR matrices R, A, B of
// Alg. 2 are never materialised.
#include <algorithm>

#include "common.cuh"
#include "gemm_dmma.cuh"
#include "mvn_internal.h"
#include "normal.cuh"

namespace mvn {
namespace sovk {
constexpr int M = 64;                    // SOV row block
constexpr int NB = 128;                  // max samples per block (= chain threads)
// K-chunk rows per pipeline stage and stages (same bytes in flight: BK * STAGES = 64); compile-time
// MVN_SOV_BK for experiments. 32 x 2 (default): half the ring handshakes of 16 x 4, measured 3.9 %
// faster at D and 2.4 % at E, equal at B / C (round-1 A/B, profiles/r01_sov_evolution.md); 8 x 8 is slower.
#ifndef MVN_SOV_BK
#define MVN_SOV_BK 32
#endif
constexpr int BK = MVN_SOV_BK, STAGES = 64 / MVN_SOV_BK;
constexpr int SA = M + 4;                // 68  == 4 (mod 16): conflict-free DMMA fragment loads
constexpr int SB = NB + 4;               // 132 == 4 (mod 16): the widest Y-history row (a block of w samples uses
                                         // w + 4, == 4 or 12 (mod 16) for w a multiple of 8: conflict-free too)
constexpr int SS = NB + 8;               // S tile stride (16-byte fragment stores conflict-free)
// GEMM warps (8; 16 warps of 16 x 32 tiles were measured slower in round 1)
constexpr int GW = 8;
constexpr int NGEMM = 32 * GW, NCHAIN = NB, NPROD = 32, NT = NGEMM + NCHAIN + NPROD;
constexpr int STAGE = BK * (SA + SB);                    // doubles per pipeline stage
constexpr int OFF_S = STAGES * STAGE;                    // S[64][SS]: s, then y, of the row block
constexpr int OFF_LD = OFF_S + M * SS;                   // Ld[64 cols][64 rows] (column-major)
constexpr int OFF_PS = OFF_LD + M * M;                   // per-row, per-chain-warp (max, sum) [64][4][2]
constexpr int OFF_AG = OFF_PS + M * 4 * 2;               // [3][64]: a, b, G (as double bits)
constexpr int OFF_DINV = OFF_AG + 3 * M;                 // [64]: 1 / L_kk of the row block
constexpr int OFF_ELL8 = OFF_DINV + M;                   // [8][NB]: log weights of the current 8-row sub-block
constexpr int OFF_P8 = OFF_ELL8 + 8 * NB;                // [8][NB]: exp(ell - c_w) of the sub-block (b = +inf path)
constexpr int OFF_BAR = OFF_P8 + 8 * NB;                 // full[STAGES], empty[STAGES] mbarriers
constexpr int SMEM = (OFF_BAR + 2 * STAGES) * 8;
constexpr int CPB = M / BK;                              // K-chunks per row block
enum : int { BAR_SFULL = 1, BAR_YREADY = 2, BAR_CHAIN = 3 };
constexpr int N_SFULL = NGEMM + NCHAIN, N_YREADY = NCHAIN + NPROD;
}  // namespace sovk

__device__ __forceinline__ void cp_async16_zfill(void *smem, const void *gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes));
}

// L2 residency: the L panel is shared by every CTA (keep it: evict_last), the Y history is private
// streaming data read once per row block (evict_first), so the L rows of the current row blocks
// survive the ~2 TB/s of Y traffic that passes through L2.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ void cp_async16_hint(void *smem, const void *gmem, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, unsigned bytes, uint64_t *bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}

__device__ __forceinline__ uint64_t lattice_shift(uint64_t seed, uint64_t r, uint64_t k) {
    // SplitMix64 output function of the counter seed + GAMMA * (r*2^32 + k + 1) (reading R8)
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * ((r << 32) + k + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double lattice_w(uint64_t j, uint64_t G, uint64_t D) {
    const uint64_t X = j * G + D;
    return ((double)(X >> 12) + 0.5) * 0x1p-52;
}

struct SovArgs {
    const double *L;
    int64_t n;
    int nrb;                  // row blocks of 64 (ceil(n/64))
    const double *a, *b;      // b may be null (+inf)
    const uint64_t *G;
    int64_t N;
    uint64_t seed;
    const int64_t *cta;       // [grid][3]: first global sample, sample count, first block index
    int64_t n_pad;            // Y-history rows per slot (nrb*64)
    double *Y;                // [grid][n_pad * SB]: per block [n_pad][w + 4] (padded for conflict-free DMMA loads)
    double *part;             // [nblk][n_pad][2]
    // soft grid lockstep (L panel reuse in L2): producer of step s = b*nrb + rb waits until every CTA
    // that has step s - lag has issued it; step_done[s] counts issuers, need[b] = CTAs with > b blocks.
    int lag;                  // 0 = off
    int *step_done;           // [max blocks][nrb]
    const int *need;          // [max blocks]
    int hints;                // L2 cache-policy hints on the producer's copies
    int serial_rb;            // row blocks rb <= serial_rb * 128 / w: GEMM of rb waits for the chain of rb-1
    int unit_mode;            // 1: blocks are the global 128-sample units (deterministic per-unit partials)
    int64_t part_stride;      // rows per block in `part` (n_pad, or n for the caller's unit partials)
    // row phases (mvn_sweep_rows): this launch runs row blocks [rb0, rb1) of every sample block; the
    // chain state that crosses row blocks is the log weight ell (ell[g - g_base] between launches)
    // and the Y history, which then needs one slot per sample block (yoff[cta]: the CTA's first slot,
    // in doubles from Y; the CTA's blocks follow at n_pad * (w + 4) each). Whole sweep: rb0 = 0,
    // rb1 = nrb, ell = yoff = null (one Y slot per CTA, reused by its blocks).
    int rb0, rb1;
    double *ell;
    int64_t g_base;
    const int64_t *yoff;
    // NEXT-3 factored update (k_sov_tlr): off-diagonal tiles of L as U_t V_t^T in slots of 128 x tkmax
    // (mvn_tlr_potrf), t = I(I-1)/2 + J, rank tranks[t]; the diagonal tiles are read from L
    const double *tU = nullptr, *tV = nullptr;
    const int *tranks = nullptr;
    int tkmax = 0;
};

// Sample blocks of a CTA: its `count` samples are split into nblk = ceil(count / 128) blocks whose
// widths are multiples of 8 (the DMMA n-dimension) spread as evenly as possible (540 -> 112, 112,
// 112, 104, 104), so no block degenerates to a sliver whose GEMM is too short to hide the chain,
// and a small per-CTA share is padded by < 8 samples (a rank's 1/8 of config D: 67.6 samples per
// CTA -> one 72-wide block; with 32-wide granularity it was 96, 29 % of the DMMA work padding).
// Block b starts at sample offset off and holds cnt <= w samples (only the last block can have
// cnt < w).
// Unit mode (a CTA's range is whole 128-sample units of the global sample index): block b is unit b
// of the range, so a unit's samples sit on the same lanes whatever the partition (W-independent
// per-unit partials).
struct BlockGeom { int64_t off; int cnt, w; };
__host__ __device__ __forceinline__ BlockGeom block_geom(int64_t count, int b, int unit_mode = 0) {
    if (unit_mode) {
        BlockGeom g;
        g.off = (int64_t)b * sovk::NB;
        const int64_t left = count - g.off;
        g.cnt = (int)(left < sovk::NB ? left : sovk::NB);
        g.w = (g.cnt + 7) & ~7;
        return g;
    }
    const int64_t units = (count + 7) / 8, nblk = (count + sovk::NB - 1) / sovk::NB;
    const int64_t q = units / nblk, r = units % nblk;
    BlockGeom g;
    g.w = (int)(8 * (q + (b < r ? 1 : 0)));
    g.off = 8 * ((int64_t)b * q + (b < r ? b : r));
    const int64_t left = count - g.off;
    g.cnt = (int)(left < g.w ? left : g.w);
    return g;
}

// Y-history slot of sample block b of this CTA (see SovArgs::yoff)
__device__ __forceinline__ double *y_slot(const SovArgs &p, int64_t count, int b) {
    if (!p.yoff) return p.Y + (int64_t)blockIdx.x * p.n_pad * sovk::SB;
    int64_t off = p.yoff[blockIdx.x];
    for (int i = 0; i < b; ++i) off += p.n_pad * (block_geom(count, i, p.unit_mode).w + 4);
    return p.Y + off;
}

// ------------------------------------------------------------------------------------ producer
// One warp streams K-chunks (BK columns of the L row panel + BK rows of the Y history) into the
// STAGES-deep ring: the L columns by cp.async (one 16-byte piece per lane per column), the Y rows by
// one TMA bulk copy. The chunk of row block r whose Y rows come from row
// block r-1 is only issued after the chain warps have published Y_{r-1} (barrier Y_READY).
__device__ __forceinline__ void sov_producer(const SovArgs &p, double *sm, int64_t count, int nblk, int lane) {
    using namespace sovk;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
    uint64_t *empty = full + STAGES;
    uint32_t q = 0;
    const uint64_t pol_L = policy_evict_last(), pol_Y = policy_evict_first();
    for (int b = 0; b < nblk; ++b) {
        const int w = block_geom(count, b, p.unit_mode).w, sbw = w + 4;    // this block's Y-history row stride
        const double *Yslot = y_slot(p, count, b);
        if (p.lag > 0 && lane == 0) atomicAdd(p.step_done + (int64_t)b * p.nrb, 1);   // row block 0: no GEMM
        for (int rb = p.rb0 > 1 ? p.rb0 : 1; rb < p.rb1; ++rb) {
            const int64_t row0 = (int64_t)rb * M;
            const int R = (int)(row0 / kTile), hh = (int)(row0 % kTile);
            if (p.lag > 0) {
                const int64_t s_wait = (int64_t)b * p.nrb + rb - p.lag;
                if (lane == 0 && s_wait >= 0) {
                    const int bw = (int)(s_wait / p.nrb);
                    const int need = p.need[bw];
                    const int *cnt = p.step_done + s_wait;
                    int v;
                    while (true) {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(cnt) : "memory");
                        if (v >= need) break;
                        __nanosleep(100);
                    }
                }
                __syncwarp();
            }
            // Y_{rb-1} must be published before the chunks that read it (c >= CPB (rb-1)). For the
            // first row blocks (rb <= serial_rb) the producer waits for it before issuing ANY chunk of
            // rb: the GEMM warps then idle (spinning, no fp64) while the chain of rb-1 runs, so the
            // chain gets the fp64 pipe to itself (7x faster per row than next to DMMA) —
            // cheaper than overlapping where the GEMM of a row block is shorter than the contended chain.
            // (the GEMM of a row block scales with the block width w; the chain does not)
            // (first row block of a later phase: Y_{rb-1} was written by the previous launch)
            const int c_sync = rb == p.rb0 ? -1 : rb * w <= p.serial_rb * NB ? 0 : CPB * (rb - 1);
            for (int c = 0; c < CPB * rb; ++c, ++q) {
                if (c == c_sync) named_sync(BAR_YREADY, N_YREADY);
                const int st = q % STAGES;
                mbar_wait(&empty[st], ((q / STAGES) & 1) ^ 1);
                const int64_t kc = (int64_t)c * BK;
                double *as = sm + st * STAGE;
                double *bs = as + BK * SA;
                // A: BK L columns x 64 rows (512 B each, 1 KB apart) by cp.async, one 16 B piece per lane
                const int T = (int)(kc / kTile), cc = (int)(kc % kTile);
                const double *Lsrc = p.L + tile_offset(R, T) + (int64_t)cc * kTile + hh + lane * 2;
                if (p.hints) {
#pragma unroll
                    for (int t = 0; t < BK; ++t) cp_async16_hint(as + t * SA + lane * 2, Lsrc + (int64_t)t * kTile, pol_L);
                } else {
#pragma unroll
                    for (int t = 0; t < BK; ++t) cp_async16(as + t * SA + lane * 2, Lsrc + (int64_t)t * kTile);
                }
                cp_async_mbar_arrive(&full[st]);
                __syncwarp();
                // B: BK Y-history rows, contiguous at the block's row stride w + 4: one TMA bulk copy
                // of only the block's columns (+4 padding), so narrow blocks stream fewer bytes
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[st], BK * sbw * 8);
                    if (p.hints) bulk_g2s_hint(bs, Yslot + kc * sbw, BK * sbw * 8, &full[st], pol_Y);
                    else bulk_g2s(bs, Yslot + kc * sbw, BK * sbw * 8, &full[st]);
                }
            }
            if (p.lag > 0 && lane == 0) atomicAdd(p.step_done + (int64_t)b * p.nrb + rb, 1);
        }
        named_sync(BAR_YREADY, N_YREADY);                     // the block's last chain is done
    }
}

// ------------------------------------------------------------------------------------ GEMM warps
// S_r (64 x w) = L[rows r, 0:64r] * Y[0:64r, block], fp64 DMMA.8x8x4 from conflict-free shared-memory
// fragments, w = 8u. Two warp layouts:
//   u = 4, 8, 12, 16 (w a multiple of 32): 2 (rows) x 4 (columns), warp tile 32 x 8*(u/4);
//   other u: 4 (rows) x 2 (column halves), warp tile 16 x 8*ceil(u/2) or 16 x 8*floor(u/2). Warp w
//     sits on scheduler w % 4 and takes row group w % 4, so each scheduler holds both halves of one
//     row group: the 2u DMMAs per k-step are the same on every scheduler for any u.
// Template arguments: LROWS = rows per warp (32 or 16), WN = 8-column fragments of this warp (0 for
// the empty half at u = 1: it still releases the ring stages).
template <int LROWS, int WN>
__device__ __forceinline__ void sov_gemm_rowblock(double *sm, int rb, int tid, int wn0, int sbw, uint32_t &q) {
    using namespace sovk;
    constexpr int WRB = LROWS / 8;
    constexpr int GR = M / LROWS;                         // row groups
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
    uint64_t *empty = full + STAGES;
    const int lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp % GR) * LROWS;
    double acc[WRB][WN > 0 ? WN : 1][2];
#pragma unroll
    for (int i = 0; i < WRB; ++i)
#pragma unroll
        for (int j = 0; j < WN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int c = 0; c < CPB * rb; ++c, ++q) {
        const int st = q % STAGES;
        mbar_wait(&full[st], (q / STAGES) & 1);
        const double *as = sm + st * STAGE;
        const double *bs = as + BK * SA;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double fa[WRB], fb[WN > 0 ? WN : 1];
            const int kr = kk + (lane & 3);
#pragma unroll
            for (int i = 0; i < WRB; ++i) fa[i] = as[kr * SA + wm0 + i * 8 + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < WN; ++j) fb[j] = bs[kr * sbw + wn0 + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < WRB; ++i)
#pragma unroll
                for (int j = 0; j < WN; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    double *S = sm + OFF_S;
#pragma unroll
    for (int i = 0; i < WRB; ++i) {
        const int row = wm0 + i * 8 + (lane >> 2);
#pragma unroll
        for (int j = 0; j < WN; ++j) {
            const int col = wn0 + j * 8 + 2 * (lane & 3);
            *reinterpret_cast<double2 *>(S + row * SS + col) = make_double2(acc[i][j][0], acc[i][j][1]);
        }
    }
}

// ------------------------------------------------------------------------------------ chain warps
// Diagonal block L[row0:+64, row0:+64] (column-major, Ld[col*64 + row]) and the limits / generators
// of the row block, by cp.async (zero-filled past n).
template <bool HAS_B>
__device__ __forceinline__ void chain_load(const SovArgs &p, double *sm, int rb, int ct) {
    using namespace sovk;
    const int64_t row0 = (int64_t)rb * M;
    const int R = (int)(row0 / kTile), hh = (int)(row0 % kTile);
    const double *Dsrc = p.L + tile_offset(R, R) + (int64_t)hh * kTile + hh;
    double *Ld = sm + OFF_LD;
#pragma unroll
    for (int qq = 0; qq < 16; ++qq) {                    // 64 cols x 64 rows = 2048 x 16 B
        const int e = qq * NCHAIN + ct;
        const int col = e >> 5, seg = e & 31;
        cp_async16(Ld + col * M + seg * 2, Dsrc + (int64_t)col * kTile + seg * 2);
    }
    double *ag = sm + OFF_AG;
    if (ct < 96) {                                       // a, b, G: 3 x 32 segments of 2 values
        const int which = ct >> 5, seg = ct & 31;
        const int64_t k = row0 + seg * 2;
        const int valid = k + 1 < p.n ? 16 : (k < p.n ? 8 : 0);
        const int64_t kk = valid ? k : 0;
        const void *src = which == 0 ? (const void *)(p.a + kk)
                                     : which == 1 ? (const void *)(HAS_B ? p.b + kk : p.a + kk) : (const void *)(p.G + kk);
        cp_async16_zfill(ag + which * M + seg * 2, src, (which == 1 && !HAS_B) ? 0 : valid);
    }
}

// Alg. 3 on one row block for sample j (thread j of the chain group). s for row li arrives in
// S[li][j] (GEMM part + in-block contributions so far) and y_li overwrites it. Sub-blocks of 8
// rows: rows inside a sub-block update each other directly (7 predicated, independent FMAs), the
// remaining rows of the block get the sub-block's 8 y values in one pass (8 FMAs per shared-memory
// read/write). After each sub-block every warp reduces (max, sum exp) of its 32 samples' log
// weights for the 8 rows at once (8 independent shuffle trees) into ps[row][warp].
template <bool HAS_B>
__device__ __forceinline__ void chain_rowblock(const SovArgs &p, double *sm, double *Yslot, int rb, int j, int cnt,
                                               int w, uint64_t r, uint64_t jl, double &ell) {
    using namespace sovk;
    const int64_t row0 = (int64_t)rb * M;
    double *S = sm + OFF_S;
    const double *Ld = sm + OFF_LD;
    double *ps = sm + OFF_PS;
    const double *a_s = sm + OFF_AG;
    const double *b_s = a_s + M;
    const uint64_t *G_s = reinterpret_cast<const uint64_t *>(a_s + 2 * M);
    const double *dinv = sm + OFF_DINV;
    double *ELL8 = sm + OFF_ELL8;
    const int lane = j & 31, cw = j >> 5;
    const bool valid = j < cnt, incol = j < w;
    const int sbw = w + 4;
    // S_0 = 0 (no GEMM for the first row block); columns j >= w of a block whose width is not a
    // multiple of 32 are outside the GEMM tile: their lanes run as invalid samples (warp-wide
    // shuffles need whole warps) on s = 0, never feeding a reduction
    if (rb == 0 || j >= w)
        for (int li = 0; li < M; ++li) S[li * SS + j] = 0.0;
#pragma unroll 1
    for (int sb = 0; sb < M / 8; ++sb) {
        const int rb0 = sb * 8;
        const int64_t left = p.n - (row0 + rb0);
        if (left <= 0) break;                             // uniform: padded rows need no y
        const int nrows = left < 8 ? (int)left : 8;
        double s = S[rb0 * SS + j];                       // row rb0: GEMM part + earlier sub-blocks
        // b = +inf path: the per-row log-sum-exp of this sub-block uses ONE warp reference c_w (the
        // warp max of ell at the sub-block start; ell never increases, so every term is <= 1) and
        // the running product pw = exp(ell - c_w) * prod q instead of 8 exps and 8 max trees. pw is
        // non-increasing along the sub-block, so the warp max of its final value bounds every row's
        // largest term from below: if it is < 2^-960 (~1e-289) some row's sum may have underflowed
        // or gone subnormal (e.g. 8 far-tail factors q ~ 1e-44, each harmless alone), and the warp
        // takes the exact per-row max/exp path below instead (reading R10: no product underflow).
        double c_w = -CUDART_INF, pw = 0.0;
        if (!HAS_B) {
            c_w = valid ? ell : -CUDART_INF;
#pragma unroll
            for (int o = 16; o; o >>= 1) c_w = fmax(c_w, __shfl_xor_sync(0xffffffffu, c_w, o));
            pw = (valid && c_w != -CUDART_INF) ? exp(ell - c_w) : 0.0;
        }
        double *P8 = sm + OFF_P8;
#pragma unroll 1
        for (int i = 0; i < nrows; ++i) {
            const int li = rb0 + i;
            const int64_t k = row0 + li;
            // next row's s without the current row's term, read before y exists (off the critical path)
            const double s_next = (i + 1 < 8) ? S[(li + 1) * SS + j] : 0.0;
            // lanes past the block's columns run a harmless central step (a' = 0): s = 0 there, and
            // a' = a / L_kk could sit in the far tail and send the whole warp down the Newton path
            const double ap = incol ? (a_s[li] - s) * dinv[li] : 0.0;
            const double wq = lattice_w(jl, G_s[li], lattice_shift(p.seed, r, (uint64_t)k));
            double lq, y;
            if (HAS_B) {
                sov_step(ap, incol ? (b_s[li] - s) * dinv[li] : CUDART_INF, wq, lq, y);
            } else {
                double q;
#ifdef MVN_SOV_FAKECHAIN   // timing experiment only: no Phi / Phi^-1 (results are wrong)
                q = 0.999; lq = -1.0005e-3; y = (wq - 0.5) + 1e-30 * ap;
#else
                sov_step_upper(ap, wq, lq, y, q);
#endif
                pw *= q;
                P8[i * NB + j] = pw;
            }
            ell += lq;
            S[li * SS + j] = y;
            ELL8[i * NB + j] = ell;
            if (incol) Yslot[k * sbw + j] = y;
            if (i + 1 < 8) s = s_next + Ld[li * M + li + 1] * y;   // row li+1 carried in a register
#pragma unroll
            for (int d = 2; d < 8; ++d)
                if (i + d < 8) S[(li + d) * SS + j] += Ld[li * M + li + d] * y;
        }
        // per-row log-sum-exp over this warp's samples, 8 rows at once
        double m[8], e[8];
        bool fast = false;
        if (!HAS_B) {
            double pmax = valid ? pw : 0.0;
#pragma unroll
            for (int o = 16; o; o >>= 1) pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
            fast = pmax >= 0x1p-960;
        }
        if (fast) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                m[i] = c_w;
                e[i] = (valid && i < nrows && c_w != -CUDART_INF) ? P8[i * NB + j] : 0.0;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) m[i] = (valid && i < nrows) ? ELL8[i * NB + j] : -CUDART_INF;
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int i = 0; i < 8; ++i) m[i] = fmax(m[i], __shfl_xor_sync(0xffffffffu, m[i], o));
#pragma unroll
            for (int i = 0; i < 8; ++i) e[i] = (valid && i < nrows && m[i] != -CUDART_INF) ? exp(ELL8[i * NB + j] - m[i]) : 0.0;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int i = 0; i < 8; ++i) e[i] += __shfl_xor_sync(0xffffffffu, e[i], o);
        if (lane < nrows) {
            double mi = m[0], ei = e[0];
#pragma unroll
            for (int i = 1; i < 8; ++i)
                if (lane == i) { mi = m[i]; ei = e[i]; }
            *reinterpret_cast<double2 *>(ps + ((rb0 + lane) * 4 + cw) * 2) = make_double2(mi, ei);
        }
        double yv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) yv[i] = S[(rb0 + i) * SS + j];
#pragma unroll 2
        for (int li = rb0 + 8; li < M; ++li) {
            double t = S[li * SS + j];
#pragma unroll
            for (int i = 0; i < 8; ++i) t += Ld[(rb0 + i) * M + li] * yv[i];
            S[li * SS + j] = t;
        }
    }
}

template <bool HAS_B>
__global__ void __launch_bounds__(sovk::NT, 1) k_sov(SovArgs p) {
    using namespace sovk;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int64_t g_first = p.cta[blockIdx.x * 3], count = p.cta[blockIdx.x * 3 + 1], blk_first = p.cta[blockIdx.x * 3 + 2];
    const int nblk = (int)((count + NB - 1) / NB);
    if (tid == 0) {
        uint64_t *full = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);                      // + 32 cp.async arrivals + bulk tx bytes
            mbar_init(&full[STAGES + s], NGEMM / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (tid < NGEMM) {
        // ============================================================ GEMM warps
        uint32_t q = 0;
        const int warp = tid >> 5;
        for (int b = 0; b < nblk; ++b) {
            const int u = block_geom(count, b, p.unit_mode).w >> 3;   // 8-column fragments of the block
            const int sbw = 8 * u + 4;                          // the block's Y-history row stride
            // layout 2 x 4 (u % 4 == 0): column group warp / 2; layout 4 x 2: half warp / 4
            const int half = warp >> 2, u0 = (u + 1) >> 1;
            const int wn0 = (u & 3) == 0 ? (warp >> 1) * 2 * u : half * 8 * u0;
            for (int rb = p.rb0 > 1 ? p.rb0 : 1; rb < p.rb1; ++rb) {
#define MVN_G2(U) case U: if (half == 0) sov_gemm_rowblock<16, (U + 1) / 2>(sm, rb, tid, wn0, sbw, q); \
                          else sov_gemm_rowblock<16, U / 2>(sm, rb, tid, wn0, sbw, q); break;
                switch (u) {
                    case 4: sov_gemm_rowblock<32, 1>(sm, rb, tid, wn0, sbw, q); break;
                    case 8: sov_gemm_rowblock<32, 2>(sm, rb, tid, wn0, sbw, q); break;
                    case 12: sov_gemm_rowblock<32, 3>(sm, rb, tid, wn0, sbw, q); break;
                    case 16: sov_gemm_rowblock<32, 4>(sm, rb, tid, wn0, sbw, q); break;
                    MVN_G2(1) MVN_G2(2) MVN_G2(3) MVN_G2(5) MVN_G2(6) MVN_G2(7) MVN_G2(9) MVN_G2(10) MVN_G2(11)
                    MVN_G2(13) MVN_G2(14) MVN_G2(15)
                    default: break;
                }
#undef MVN_G2
                named_arrive(BAR_SFULL, N_SFULL);
            }
        }
    } else if (tid < NGEMM + NCHAIN) {
        // ============================================================ chain warps
        const int j = tid - NGEMM;
        for (int b = 0; b < nblk; ++b) {
            const BlockGeom bg = block_geom(count, b, p.unit_mode);
            const int64_t g0 = g_first + bg.off;
            const int cnt = bg.cnt;
            const int w = bg.w;
            const uint64_t g = (uint64_t)(g0 + (j < cnt ? j : 0));
            const uint64_t r = g / (uint64_t)p.N;
            const uint64_t jl = g - r * (uint64_t)p.N + 1ull;    // 1-based lattice index
            const int64_t blk = blk_first + b;
            double *Yslot = y_slot(p, count, b);
            double ell = (p.ell && p.rb0 > 0 && j < cnt) ? p.ell[g - p.g_base] : 0.0;
            for (int rb = p.rb0; rb < p.rb1; ++rb) {
                chain_load<HAS_B>(p, sm, rb, j);                  // Ld / a / G of this row block
                cp_async_commit();
                if (rb > 0) named_sync(BAR_SFULL, N_SFULL);       // S_rb written by the GEMM warps
                cp_async_wait<0>();
                named_sync(BAR_CHAIN, NCHAIN);
                if (j < M) sm[OFF_DINV + j] = 1.0 / sm[OFF_LD + j * M + j];
                named_sync(BAR_CHAIN, NCHAIN);
                if (j < ((w + 31) & ~31)) chain_rowblock<HAS_B>(p, sm, Yslot, rb, j, cnt, w, r, jl, ell);
                __threadfence();                                  // Y_rb: generic-proxy writes ...
                asm volatile("fence.proxy.async.global;\n" ::: "memory");   // ... visible to the TMA reads
                named_arrive(BAR_YREADY, N_YREADY);
                named_sync(BAR_CHAIN, NCHAIN);                   // ps complete, Ld / S free
                if (j < M) {
                    const int64_t k = (int64_t)rb * M + j;
                    if (k < p.n) {
                        const double *ps = sm + OFF_PS + j * 8;
                        const int nw = (w + 31) >> 5;
                        double mm = -CUDART_INF;
                        for (int qq = 0; qq < nw; ++qq) mm = fmax(mm, ps[2 * qq]);
                        double ss = 0.0;
                        if (mm != -CUDART_INF)
                            for (int qq = 0; qq < nw; ++qq)
                                if (ps[2 * qq] != -CUDART_INF) ss += ps[2 * qq + 1] * exp(ps[2 * qq] - mm);
                        *reinterpret_cast<double2 *>(p.part + (blk * p.part_stride + k) * 2) = make_double2(mm, ss);
                    }
                }
            }
            if (p.ell && j < cnt) p.ell[(int64_t)g - p.g_base] = ell;   // for the next row phase
        }
    } else {
        // ============================================================ producer warp
        sov_producer(p, sm, count, nblk, tid & 31);
    }
}

// ------------------------------------------------------------------------------------ NEXT-3
// k_sov_tlr: the sweep with the SOV update in factored form, s_k = sum_J U_TJ (V_TJ^T Y_J) over the
// tiles J < T of the row's tile row T ("factored SOV update A -= U(V^T Y)";
// the paper itself keeps (b)-(d) dense, which k_sov on the reconstructed L~ does). Same
// samples, lattice, chain (chain_load / chain_rowblock) and partials as k_sov; the GEMM warps run
// per 64-row block rb (tile row T = rb / 2, half h = rb % 2):
//   for each J < T with rank r: W = V_TJ(:, c0:c0+64)^T Y_J (<= 64 x w, K = 128, Y_J staged in
//   shared memory), acc += U_TJ(64h:64h+64, c0:c0+64) W; for h = 1 also the dense part of the
//   diagonal tile, acc += L_TT(64:128, 0:64) Y_T(0:64).
// The GEMM of rb starts after the chain of rb - 1 (no overlap: the S tile is the accumulator, which
// keeps one fragment array per thread live). No producer warp: the operands come from L2 (U, V: direct fragment loads; Y: staged, ld.global.cg since the CTA's Y slot is rewritten
// by every sample block). Flops per (sample, tile): 2 x (2 128 r) + 2 64 r x 2 halves, vs 2 128^2
// dense: the factored form pays when r < ~43.
namespace sovt {
constexpr int NG = sovk::NGEMM, NTH = NG + sovk::NCHAIN;  // 8 GEMM warps + 4 chain warps, no producer
constexpr int BAR_G = 4;                                   // the GEMM warps' staging barrier
constexpr int SW = sovk::NB + 4;                           // W / staged-Y row stride (== 4 mod 16)
constexpr int OFF_W = 0, OFF_BS = OFF_W + 64 * SW;         // inside k_sov's ring region (unused here)
static_assert(OFF_BS + 2 * 16 * SW <= sovk::OFF_S, "TLR staging (W + two B buffers) must fit the ring region");
}  // namespace sovt

// acc(8 rows of warp wp x w) += A(8 x K) * B(K x w): A fragments straight from global (a(m, k) =
// A[m * am + k * ak], m = the warp's row 8 wp + lane / 4), B rows staged 16 at a time from the Y
// history (rows y0 + k, stride sbw, `cg` loads) or read from the W tile in shared memory.
template <int NF>
__device__ __forceinline__ void tlr_rows_gemm(double (&acc)[16][2], const double *__restrict__ A, int64_t am, int64_t ak,
                                              int K, const double *Y, int64_t y0, int sbw, const double *Wsm,
                                              double *BS, int w, int tid) {
    using namespace sovt;
    const int lane = tid & 31, wp = tid >> 5;
    const int mrow = 8 * wp + (lane >> 2);
    // the next chunk's A fragments (4 per lane) are loaded into registers and the next chunk's B rows
    // copied into the other half of a double-buffered BS by cp.async (16-byte pieces, zero-filled
    // past K) while the current chunk's DMMAs run; one barrier per chunk
    double aN[4];
    auto loadA = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int kr = 4 * q + (lane & 3);
            aN[q] = (k0 + kr < K) ? __ldg(A + (int64_t)mrow * am + (int64_t)(k0 + kr) * ak) : 0.0;
        }
    };
    const int hw = w >> 1;                                // 16-byte pieces per staged row
    auto issueB = [&](int k0, double *buf) {
        for (int e = tid; e < 16 * hw; e += NG) {
            const int kk = e / hw, pc = e - kk * hw;
            const bool in = k0 + kk < K;
            cp_async16_zfill(buf + kk * SW + 2 * pc, in ? Y + (y0 + k0 + kk) * sbw + 2 * pc : Y, in ? 16 : 0);
        }
        cp_async_commit();
    };
    loadA(0);
    if (Y) {
        named_sync(BAR_G, NG);                            // the previous users of both BS buffers are done
        issueB(0, BS);
    }
    for (int k0 = 0, c = 0; k0 < K; k0 += 16, ++c) {
        double a[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) a[q] = aN[q];
        const double *Bs;
        if (Y) {
            cp_async_wait<0>();
            named_sync(BAR_G, NG);                        // chunk c landed; chunk c - 1's readers are done
            if (k0 + 16 < K) issueB(k0 + 16, BS + ((c + 1) & 1) * 16 * SW);
            Bs = BS + (c & 1) * 16 * SW;
        } else {
            Bs = Wsm + (int64_t)k0 * SW;
        }
        if (k0 + 16 < K) loadA(k0 + 16);
#pragma unroll
        for (int kk = 0; kk < 16; kk += 4) {
            const int kr = kk + (lane & 3);
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const double b = Bs[kr * SW + 8 * f + (lane >> 2)];
                dmma(acc[f][0], acc[f][1], a[kk >> 2], b);
            }
        }
    }
}

// S(8 rows of warp wp, :) += acc (the warp's own fragments of the S tile)
template <int NF>
__device__ __forceinline__ void tlr_add_to_s(double *sm, const double (&acc)[16][2], int tid) {
    double *S = sm + sovk::OFF_S;
    const int lane = tid & 31, m = 8 * (tid >> 5) + (lane >> 2);
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        double2 *d = reinterpret_cast<double2 *>(S + m * sovk::SS + 8 * f + 2 * (lane & 3));
        const double2 v = *d;
        *d = make_double2(v.x + acc[f][0], v.y + acc[f][1]);
    }
}

template <int NF>
__device__ __forceinline__ void tlr_tile_term(const SovArgs &p, double *sm, const double *Yslot, int sbw, int T, int J,
                                              int h, int w, int tid) {
    using namespace sovt;
    const int64_t t = (int64_t)T * (T - 1) / 2 + J;
    const int r = p.tranks[t];
    const double *U = p.tU + t * 128 * (int64_t)p.tkmax, *V = p.tV + t * 128 * (int64_t)p.tkmax;
    double *Wsm = sm + OFF_W, *BS = sm + OFF_BS;
    const int lane = tid & 31, wp = tid >> 5;
    for (int c0 = 0; c0 < r; c0 += 64) {
        const int rc = r - c0 < 64 ? r - c0 : 64;
        double acc[16][2];
        // W (rc x w) = V(:, c0 + m)^T Y_J: a(m, k) = V[(c0 + m) 128 + k]; rows m >= rc are not read
        // (a warp's rows past rc compute garbage-free zeros: its A pointer is clamped, the rows dropped)
#pragma unroll
        for (int f = 0; f < 16; ++f) acc[f][0] = acc[f][1] = 0.0;
        const int mrow = 8 * wp + (lane >> 2);
        const double *Vw = V + (int64_t)c0 * 128 + (mrow < rc ? 0 : -(int64_t)mrow * 128);   // row m -> column c0 + m (clamped to c0)
        tlr_rows_gemm<NF>(acc, Vw, 128, 1, 128, Yslot, (int64_t)J * 128, sbw, nullptr, BS, w, tid);
        named_sync(BAR_G, NG);                            // the previous W's readers are done
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const int col = 8 * f + 2 * (lane & 3);
            const bool ok = mrow < rc;
            Wsm[mrow * SW + col] = ok ? acc[f][0] : 0.0;
            Wsm[mrow * SW + col + 1] = ok ? acc[f][1] : 0.0;
        }
        named_sync(BAR_G, NG);
        // S(64h + m, :) += U(64h + m, c0 + k) W(k, :), k < rc
#pragma unroll
        for (int f = 0; f < 16; ++f) acc[f][0] = acc[f][1] = 0.0;
        tlr_rows_gemm<NF>(acc, U + (int64_t)c0 * 128 + 64 * h, 1, 128, rc, nullptr, 0, 0, Wsm, BS, w, tid);
        tlr_add_to_s<NF>(sm, acc, tid);
    }
}

template <int NF>
__device__ __forceinline__ void tlr_gemm_rowblock(const SovArgs &p, double *sm, const double *Yslot, int sbw, int rb,
                                                  int w, int tid) {
    using namespace sovt;
    const int T = rb >> 1, h = rb & 1;
    named_sync(sovk::BAR_YREADY, NTH);                    // chain(rb - 1) done: Y rows of rb - 1, S free
    {
        double *S = sm + sovk::OFF_S;
        const int lane = tid & 31, m = 8 * (tid >> 5) + (lane >> 2);
#pragma unroll
        for (int f = 0; f < NF; ++f)
            *reinterpret_cast<double2 *>(S + m * sovk::SS + 8 * f + 2 * (lane & 3)) = make_double2(0.0, 0.0);
    }
    for (int J = 0; J < T; ++J) tlr_tile_term<NF>(p, sm, Yslot, sbw, T, J, h, w, tid);
    if (h == 1) {                                         // dense part of the diagonal tile: L_TT(64:, 0:64) Y_T(0:64)
        double acc[16][2];
#pragma unroll
        for (int f = 0; f < 16; ++f) acc[f][0] = acc[f][1] = 0.0;
        const double *Ltt = p.L + tile_offset(T, T) + 64;
        tlr_rows_gemm<NF>(acc, Ltt, 1, 128, 64, Yslot, (int64_t)T * 128, sbw, nullptr, sm + OFF_BS, w, tid);
        tlr_add_to_s<NF>(sm, acc, tid);
    }
    named_arrive(sovk::BAR_SFULL, NTH);
}

template <bool HAS_B>
__global__ void __launch_bounds__(sovt::NTH, 1) k_sov_tlr(SovArgs p) {
    using namespace sovk;
    extern __shared__ double sm[];
    const int tid = threadIdx.x;
    const int64_t g_first = p.cta[blockIdx.x * 3], count = p.cta[blockIdx.x * 3 + 1], blk_first = p.cta[blockIdx.x * 3 + 2];
    const int nblk = (int)((count + NB - 1) / NB);
    if (tid < NGEMM) {
        // ============================================================ GEMM warps (factored update)
        for (int b = 0; b < nblk; ++b) {
            const int w = block_geom(count, b, p.unit_mode).w, sbw = w + 4;
            const double *Yslot = y_slot(p, count, b);
            for (int rb = 1; rb < p.nrb; ++rb) {
#define MVN_TG(F) case F: tlr_gemm_rowblock<F>(p, sm, Yslot, sbw, rb, w, tid); break;
                switch (w >> 3) {
                    MVN_TG(1) MVN_TG(2) MVN_TG(3) MVN_TG(4) MVN_TG(5) MVN_TG(6) MVN_TG(7) MVN_TG(8)
                    MVN_TG(9) MVN_TG(10) MVN_TG(11) MVN_TG(12) MVN_TG(13) MVN_TG(14) MVN_TG(15) MVN_TG(16)
                    default: break;
                }
#undef MVN_TG
            }
            named_sync(BAR_YREADY, sovt::NTH);            // the block's last chain is done (balances its arrival)
        }
    } else {
        // ============================================================ chain warps (as k_sov)
        const int j = tid - NGEMM;
        for (int b = 0; b < nblk; ++b) {
            const BlockGeom bg = block_geom(count, b, p.unit_mode);
            const int64_t g0 = g_first + bg.off;
            const int cnt = bg.cnt;
            const int w = bg.w;
            const uint64_t g = (uint64_t)(g0 + (j < cnt ? j : 0));
            const uint64_t r = g / (uint64_t)p.N;
            const uint64_t jl = g - r * (uint64_t)p.N + 1ull;
            const int64_t blk = blk_first + b;
            double *Yslot = y_slot(p, count, b);
            double ell = 0.0;
            for (int rb = 0; rb < p.nrb; ++rb) {
                chain_load<HAS_B>(p, sm, rb, j);
                cp_async_commit();
                if (rb > 0) named_sync(BAR_SFULL, sovt::NTH);
                cp_async_wait<0>();
                named_sync(BAR_CHAIN, NCHAIN);
                if (j < M) sm[OFF_DINV + j] = 1.0 / sm[OFF_LD + j * M + j];
                named_sync(BAR_CHAIN, NCHAIN);
                if (j < ((w + 31) & ~31)) chain_rowblock<HAS_B>(p, sm, Yslot, rb, j, cnt, w, r, jl, ell);
                __threadfence();
                named_arrive(BAR_YREADY, sovt::NTH);
                named_sync(BAR_CHAIN, NCHAIN);
                if (j < M) {
                    const int64_t k = (int64_t)rb * M + j;
                    if (k < p.n) {
                        const double *ps = sm + OFF_PS + j * 8;
                        const int nw = (w + 31) >> 5;
                        double mm = -CUDART_INF;
                        for (int qq = 0; qq < nw; ++qq) mm = fmax(mm, ps[2 * qq]);
                        double ss = 0.0;
                        if (mm != -CUDART_INF)
                            for (int qq = 0; qq < nw; ++qq)
                                if (ps[2 * qq] != -CUDART_INF) ss += ps[2 * qq + 1] * exp(ps[2 * qq] - mm);
                        *reinterpret_cast<double2 *>(p.part + (blk * p.part_stride + k) * 2) = make_double2(mm, ss);
                    }
                }
            }
        }
    }
}

// K6: combine block partials per prefix in a fixed order (deterministic for a given nblk). A CTA
// takes 32 prefixes (lane = prefix: 512-byte coalesced reads of the (max, sum) pairs) and RS
// contiguous slices of the blocks (threadIdx.y); each thread combines its slice in ascending block
// order, then lane-wise one warp combines the RS slice results in ascending slice order. One thread
// per prefix looping over all ~890 blocks was 0.50 ms of config A's 4.7 ms step
// (profiles/r02_sov_A_ncu.md).
constexpr int RS = 16;
__global__ void __launch_bounds__(32 * RS)
k_reduce_blocks(const double *__restrict__ part, int64_t nblk, int64_t n, int64_t n_pad,
                double *__restrict__ Mo, double *__restrict__ So) {
    __shared__ double sm[RS][32], ss[RS][32];
    const int lane = threadIdx.x, j = threadIdx.y;
    const int64_t k = blockIdx.x * (int64_t)32 + lane;
    const int64_t per = (nblk + RS - 1) / RS, b0 = j * per, b1 = b0 + per < nblk ? b0 + per : nblk;
    double m = -CUDART_INF, s = 0.0;
    if (k < n) {
        const double2 *p = reinterpret_cast<const double2 *>(part) + k;
#pragma unroll 4
        for (int64_t b = b0; b < b1; ++b) m = fmax(m, p[b * n_pad].x);
        if (m != -CUDART_INF) {
#pragma unroll 4
            for (int64_t b = b0; b < b1; ++b) {
                const double2 v = p[b * n_pad];
                if (v.x != -CUDART_INF) s += v.y * exp(v.x - m);
            }
        }
    }
    sm[j][lane] = m;
    ss[j][lane] = s;
    __syncthreads();
    if (j != 0 || k >= n) return;
    double mm = -CUDART_INF;
#pragma unroll
    for (int q = 0; q < RS; ++q) mm = fmax(mm, sm[q][lane]);
    double t = 0.0;
    if (mm != -CUDART_INF) {
#pragma unroll
        for (int q = 0; q < RS; ++q)
            if (sm[q][lane] != -CUDART_INF) t += ss[q][lane] * exp(sm[q][lane] - mm);
    }
    Mo[k] = mm;
    So[k] = t;
}

// The caller's per-unit partials (mvn_prefix_reduce): one thread per prefix, strictly ascending unit
// order, (-inf, 0) units skipped, so the bits do not depend on how the units were split over ranks
// or padded (SURVEY 8(e)'s deterministic combine; parallel.combine_units_deterministic).
__global__ void k_reduce_units(const double *__restrict__ part, int64_t units, int64_t n,
                               double *__restrict__ Mo, double *__restrict__ So) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    double m = -CUDART_INF;
    for (int64_t b = 0; b < units; ++b) m = fmax(m, part[(b * n + k) * 2]);
    double s = 0.0;
    if (m != -CUDART_INF)
        for (int64_t b = 0; b < units; ++b) {
            const double mb = part[(b * n + k) * 2], sb = part[(b * n + k) * 2 + 1];
            if (mb != -CUDART_INF) s += sb * exp(mb - m);
        }
    Mo[k] = m;
    So[k] = s;
}

cudaError_t sov_init() {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_sov<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sovk::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_sov<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sovk::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_sov_tlr<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sovk::SMEM))) return e;
    if ((e = cudaFuncSetAttribute(k_sov_tlr<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sovk::SMEM))) return e;
    return cudaSuccess;
}

int sov_block_samples() { return sovk::NB; }
int sov_y_stride() { return sovk::SB; }

// Unit mode: the global units [u0, u1) of 128 samples (the last one clipped at g_end) over `grid`
// CTAs, floor/ceil(units / grid) whole units each; block index = unit - u0.
int64_t sov_partition_units(int64_t u0, int64_t u1, int64_t g_end, int grid, int64_t *cta) {
    const int64_t nu = u1 - u0, base = nu / grid, rem = nu % grid;
    int64_t u = u0;
    for (int c = 0; c < grid; ++c) {
        const int64_t k = base + (c < rem ? 1 : 0);
        const int64_t g = u * sovk::NB, ge = std::min<int64_t>((u + k) * sovk::NB, g_end);
        cta[3 * c] = g;
        cta[3 * c + 1] = k > 0 ? ge - g : 0;
        cta[3 * c + 2] = u - u0;
        u += k;
    }
    return nu;
}

// Balanced partition of [g_begin, g_end) over `grid` CTAs: CTA c gets a contiguous share of
// floor/ceil(nsamp/grid) samples, processed as blocks of 128 (last one narrowed to 32k).
int64_t sov_partition(int64_t g_begin, int64_t g_end, int grid, int64_t *cta) {
    const int64_t ns = g_end - g_begin, base = ns / grid, rem = ns % grid;
    int64_t blk = 0, g = g_begin;
    for (int c = 0; c < grid; ++c) {
        const int64_t cnt = base + (c < rem ? 1 : 0);
        cta[3 * c] = g;
        cta[3 * c + 1] = cnt;
        cta[3 * c + 2] = blk;
        g += cnt;
        blk += (cnt + sovk::NB - 1) / sovk::NB;
    }
    return blk;
}

// Row phases: Y slot offsets (doubles) of each CTA's first sample block, one slot of n_pad x (w + 4)
// per block (block_geom widths); returns the total doubles.
int64_t sov_phase_yoff(const int64_t *cta, int grid, int64_t n_pad, int unit_mode, int64_t *yoff) {
    int64_t off = 0;
    for (int c = 0; c < grid; ++c) {
        yoff[c] = off;
        const int64_t count = cta[3 * c + 1];
        const int nb = (int)((count + sovk::NB - 1) / sovk::NB);
        for (int b = 0; b < nb; ++b) off += n_pad * (block_geom(count, b, unit_mode).w + 4);
    }
    return off;
}

cudaError_t launch_sov(const SovLaunch &L, cudaStream_t st) {
    SovArgs a;
    a.L = L.L; a.n = L.n; a.nrb = (int)((L.n + 63) / 64); a.a = L.a; a.b = L.b; a.G = L.G; a.N = L.N;
    a.seed = L.seed; a.cta = L.cta; a.n_pad = (int64_t)a.nrb * 64; a.Y = L.Y; a.part = L.part;
    a.lag = L.lag; a.step_done = L.step_done; a.need = L.need; a.hints = L.hints; a.serial_rb = L.serial_rb;
    a.unit_mode = L.unit_mode; a.part_stride = L.unit_mode ? L.n : a.n_pad;
    a.rb0 = L.rb1 > 0 ? L.rb0 : 0; a.rb1 = L.rb1 > 0 ? L.rb1 : a.nrb; a.ell = L.ell; a.g_base = L.g_begin; a.yoff = L.yoff;
    if (a.lag > 0) {
        cudaError_t e = cudaMemsetAsync(L.step_done, 0, sizeof(int) * (size_t)L.max_blocks * a.nrb, st);
        if (e != cudaSuccess) return e;
    }
    a.tU = L.tU; a.tV = L.tV; a.tranks = L.tranks; a.tkmax = L.tkmax;
    if (L.tU) {                                          // NEXT-3 factored update (whole sweeps only)
        if (L.rb1 > 0 || L.lag > 0) return cudaErrorInvalidValue;
        if (L.b) k_sov_tlr<true><<<L.grid, sovt::NTH, sovk::SMEM, st>>>(a);
        else k_sov_tlr<false><<<L.grid, sovt::NTH, sovk::SMEM, st>>>(a);
    } else if (L.b) k_sov<true><<<L.grid, sovk::NT, sovk::SMEM, st>>>(a);
    else k_sov<false><<<L.grid, sovk::NT, sovk::SMEM, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (L.unit_mode || L.rb1 > 0) return cudaSuccess;          // the caller reduces the partials
    return launch_reduce_blocks(L.part, L.nblk, L.n, a.n_pad, L.Mout, L.Sout, st);
}

cudaError_t launch_reduce_blocks(const double *part, int64_t nblk, int64_t n, int64_t n_pad, double *M, double *S,
                                 cudaStream_t st) {
    k_reduce_blocks<<<(unsigned)((n + 31) / 32), dim3(32, RS), 0, st>>>(part, nblk, n, n_pad, M, S);
    return cudaGetLastError();
}

cudaError_t launch_reduce_units(const double *part, int64_t units, int64_t n, double *M, double *S, cudaStream_t st) {
    k_reduce_units<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(part, units, n, M, S);
    return cudaGetLastError();
}

}  // namespace mvn
