// NEXT-2 on the 5th-generation tensor cores: the MC-validation product X = L Z (fp64 accurate)
// emulated with exact int8 x int8 -> int32 tcgen05.mma (kind::i8, accumulators in TMEM) — an
// Ozaki-style split (the paper's stated future work: "mixed-precision ... tensor core execution",
// P:666). Same result contract as k_mc_trmm (first failing row per draw).
//
//   L_kt = 2^{e_k} * sum_{p=1..S} a_p(k,t) 2^{-7p},   |L_kt| <= 2^{e_k - 1}   (per-row exponent)
//   z_tj = 2^{4}   * sum_{q=1..S} b_q(t,j) 2^{-7q},   |z| <= 8.3 < 2^3      (fixed exponent)
//   a_p, b_q integers in [-64, 64] (b_1 in [-67, 67]), exact: each slice is rint of the exact
//   scaled residual, the residual after S slices (< 2^{-7S-1}) is dropped.
//   X_kj = 2^{e_k + 4} sum_{d=2}^{S+1} 2^{-7d} sum_{p+q=d} (A_p B_q)_kj      (pairs p+q <= S+1)
// Every (A_p B_q) is an exact int8 GEMM; the pairs of one level d accumulate in one int32 TMEM
// accumulator (|level sum| <= (d-1) * K * 67 * 64 < 2^31 for K <= 16,384 per flush); the epilogue
// warps flush the S levels into fp64 registers (exact int32 -> fp64, power-of-two scales).
// Dropped terms (p+q > S+1): <= S * K * 64^2 * 2^{-7(S+2)} relative to 2^{e_k+4} (1e-12 at S = 8,
// K = 65,536) — far below the 1e-9 decision margin of the parity bar.
//
// Kernel layout (one CTA per SM, persistent over items (row tile i, 64-draw block), heaviest first):
//   warps 0-3: epilogue (TMEM lanes 0-127 = the 128 rows of the tile), warp 4: TMA producer
//   (two bulk copies per 32-wide K chunk: all S slices of A (32 KB) and of B (16 KB), pre-arranged
//   in HBM in the canonical no-swizzle K-major core-matrix order), warp 5: MMA issuer (one lane,
//   S(S+1)/2 = 36 tcgen05.mma M128 N64 K32 per chunk). 4-stage smem ring with full/empty
//   mbarriers, tmem_full / tmem_empty mbarriers between the MMA issuer and the epilogue.
#include <algorithm>
#include <climits>

#include "common.cuh"
#include "mvn_internal.h"
#include "normal.cuh"
#include "umma.cuh"

namespace mvn {
namespace oz {
constexpr int S = 8;                        // slices (7 bits each)
constexpr int NS = 64;                      // draws per item (MMA N)
constexpr int KC = 32;                      // K per chunk (= one MMA K)
constexpr int A_SLICE = kTile * KC;         // 4 KB: 128 rows x 32 K-bytes
constexpr int B_SLICE = NS * KC;            // 2 KB
constexpr int A_BYTES = S * A_SLICE, B_BYTES = S * B_SLICE;
constexpr int STAGE = A_BYTES + B_BYTES;    // 48 KB
constexpr int STAGES = 4;
constexpr int FLUSH = 512;                  // chunks per TMEM flush (K = 16,384)
constexpr int NT = 192;
constexpr int SMEM = STAGES * STAGE + 1024; // + barriers / bookkeeping
constexpr uint32_t TMEM_COLS = 512;         // S levels x 64 columns
}  // namespace oz

constexpr uint32_t oz_idesc() {   // kind::i8: D s32, A/B signed, K-major, N = 64, M = 128
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(oz::NS >> 3) << 17) | ((uint32_t)(kTile >> 4) << 24);
}


__device__ __forceinline__ void oz_split(double v, int8_t *out, int stride) {
    // v in [-0.53, 0.53]: S signed 7-bit digits, exact (see header)
#pragma unroll
    for (int p = 0; p < oz::S; ++p) {
        v *= 128.0;
        const double t = rint(v);
        out[p * stride] = (int8_t)(int)t;
        v -= t;
    }
}

// Per-row power-of-two scale: rowscale[k] = 2^{e_k} with max_t |L_kt| <= 2^{e_k - 1}.
__global__ void k_oz_rowscale(const double *__restrict__ tiles, int64_t n, int nt, double *__restrict__ rowscale) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= (int64_t)nt * kTile) return;
    const int I = (int)(k / kTile), r = (int)(k % kTile);
    double m = 0.0;
    for (int J = 0; J <= I; ++J) {
        const double *T = tiles + tile_offset(I, J) + r;
        const int cols = (J == I) ? r + 1 : kTile;
        for (int c = 0; c < cols; ++c) m = fmax(m, fabs(T[(int64_t)c * kTile]));
    }
    int e;
    frexp(m, &e);                       // m < 2^e
    rowscale[k] = (m > 0.0) ? ldexp(1.0, e + 1) : 1.0;
}

// A slices: LA[(2 i (i+1) + c) * A_BYTES + p * A_SLICE + core(row, kk)] = a_p(i*128 + row, 32 c + kk).
// One thread per (row, 32-wide chunk): reads 32 consecutive L entries of the row (a column segment
// of the column-major tile is not contiguous in the row, so the reads are strided; fine for a
// one-off O(n^2) pass).
__global__ void k_oz_lslice(const double *__restrict__ tiles, int nt, const double *__restrict__ rowscale, int8_t *__restrict__ LA) {
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // over (i, c, row)
    const int64_t total_chunks = 2ll * nt * (nt + 1);
    const int64_t chunk = gid / kTile;
    if (chunk >= total_chunks) return;
    const int row = (int)(gid % kTile);
    int i = (int)((sqrt(2.0 * (double)chunk + 1.0) - 1.0) * 0.5);
    while (2ll * i * (i + 1) > chunk) --i;
    while (2ll * (i + 1) * (i + 2) <= chunk) ++i;
    const int c = (int)(chunk - 2ll * i * (i + 1));
    const int J = c >> 2, col0 = (c & 3) * oz::KC;
    const double *T = tiles + tile_offset(i, J) + row;
    const double inv = 1.0 / rowscale[(int64_t)i * kTile + row];
    int8_t *dst = LA + chunk * oz::A_BYTES;
    for (int kk = 0; kk < oz::KC; ++kk) {
        const double v = T[(int64_t)(col0 + kk) * kTile] * inv;   // exact (power-of-two scale)
        oz_split(v, dst + oz_core(row, kk), oz::A_SLICE);
    }
}

__device__ __forceinline__ uint64_t oz_mix(uint64_t seed, uint64_t s, uint64_t k) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * ((s << 32) + k + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// B slices of draws s0 .. s0+ns-1: ZB[(blk * nchunk + c) * B_BYTES + q * B_SLICE + core(j, kk)]
// = b_q(row 32 c + kk, draw blk*64 + j); rows >= n and draws >= ns are 0. z as in k_mc_gen (R20).
template <int NSB>
__global__ void k_oz_zgen(int8_t *__restrict__ ZB, int64_t n, int nchunk, int64_t s0, int64_t ns, uint64_t seed, int64_t total) {
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // over (blk, c, kk, j)
    if (gid >= total) return;
    const int j = (int)(gid % NSB);
    const int kk = (int)((gid / NSB) & 31);
    const int64_t bc = gid / (NSB * 32);                                  // blk * nchunk + c
    const int64_t blk = bc / nchunk, c = bc % nchunk;
    const int64_t k = c * oz::KC + kk, s = blk * NSB + j;
    double z = 0.0;
    if (k < n && s < ns) {
        const uint64_t X = oz_mix(seed, (uint64_t)(s0 + s), (uint64_t)k);
        const double w = ((double)(X >> 12) + 0.5) * 0x1p-52;
        z = (w <= 0.5) ? Phi_inv_lower(w) : -Phi_inv_lower(1.0 - w);
    }
    oz_split(z * 0.0625, ZB + bc * (oz::S * NSB * oz::KC) + oz_core(j, kk), NSB * oz::KC);
}

__device__ __forceinline__ void oz_mbar_wait(uint64_t *bar, uint32_t parity) { mbar_wait(bar, parity); }

// CL = 2: the two CTAs of a cluster work on the same row tile (draw blocks 2b, 2b+1) in lockstep
// and each fetches half of the shared L-slice chunk with a multicast bulk copy into BOTH CTAs'
// rings (L2 -> SM traffic for A halved); each CTA's MMA completion is committed to both CTAs'
// `empty` barriers, so a slot is refilled only when both have consumed it.

template <int CL>
__global__ void __launch_bounds__(oz::NT, 1) k_oz_trmm(const int8_t *__restrict__ LA, const int8_t *__restrict__ ZB, int64_t n,
                                                      int nt, int nblk, int64_t ns, const double *__restrict__ rowscale,
                                                      const double *__restrict__ a, int *__restrict__ first) {
    using namespace oz;
    extern __shared__ __align__(1024) uint8_t smo[];
    uint8_t *ring = smo;
    uint64_t *full = reinterpret_cast<uint64_t *>(smo + STAGES * STAGE);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;           // MMA -> epilogue (flush ready)
    uint64_t *tempty = tfull + 1;               // epilogue -> MMA (accumulators drained)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nchunk_all = nt * 4;              // chunks of 32 rows over n_pad (B layout)
    // items: (row tile, group of CL draw blocks); this CTA takes block CL * g + crank of the group
    const int crank = CL > 1 ? (int)cluster_rank() : 0;
    const int64_t nitems = (int64_t)nt * (nblk / CL);
    const int64_t item0 = blockIdx.x / CL, istep = gridDim.x / CL;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CL); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 4);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)), "n"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (CL > 1) cluster_sync_all();             // the peer's barriers exist before any multicast / remote arrive
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;
    const int nbg = nblk / CL;

    if (warp == 4) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t q = 0;
            for (int64_t item = item0; item < nitems; item += istep) {
                const int i = nt - 1 - (int)(item / nbg), blk = (int)(item % nbg) * CL + crank;
                const int nch = 4 * (i + 1);
                const int8_t *Ai = LA + 2ll * i * (i + 1) * A_BYTES;
                const int8_t *Bb = ZB + (int64_t)blk * nchunk_all * B_BYTES;
                for (int c = 0; c < nch; ++c, ++q) {
                    const int st = q % STAGES;
                    oz_mbar_wait(&empty[st], ((q / STAGES) & 1) ^ 1);
                    uint8_t *dst = ring + st * STAGE;
                    mbar_arrive_expect_tx(&full[st], STAGE);
                    if (CL == 1) {
                        bulk_g2s(dst, Ai + (int64_t)c * A_BYTES, A_BYTES, &full[st]);
                    } else {                             // my half of the A chunk, into both CTAs
                        constexpr int H = A_BYTES / CL;
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                                     " [%0], [%1], %2, [%3], %4;\n"
                                     ::"r"(smem_u32(dst + crank * H)), "l"(Ai + (int64_t)c * A_BYTES + crank * H), "r"(H),
                                       "r"(smem_u32(&full[st])), "h"((uint16_t)((1u << CL) - 1)) : "memory");
                    }
                    bulk_g2s(dst + A_BYTES, Bb + (int64_t)c * B_BYTES, B_BYTES, &full[st]);
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        uint32_t q = 0, flush = 0;
        constexpr uint32_t idesc = oz_idesc();
        for (int64_t item = item0; item < nitems; item += istep) {
            const int i = nt - 1 - (int)(item / nbg);
            const int nch = 4 * (i + 1);
            for (int c = 0; c < nch; ++c, ++q) {
                const bool fresh = (c % FLUSH) == 0;          // first chunk after a flush: overwrite TMEM
                if (fresh) {
                    oz_mbar_wait(tempty, (flush & 1) ^ 1);    // previous flush drained by the epilogue
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                }
                const int st = q % STAGES;
                oz_mbar_wait(&full[st], (q / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(ring + st * STAGE), b0 = a0 + A_BYTES;
#pragma unroll
                    for (int d = 0; d < S; ++d) {             // level d: pairs p + q = d + 2 (1-based)
#pragma unroll
                        for (int p = 0; p <= d; ++p) {
                            const int qq = d - p;
                            const uint64_t da = oz_desc(a0 + p * A_SLICE), db = oz_desc(b0 + qq * B_SLICE);
                            const uint32_t acc = (fresh && p == 0) ? 0u : 1u;
                            asm volatile("{\n .reg .pred pp;\n setp.ne.u32 pp, %4, 0;\n"
                                         " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp;\n}\n"
                                         ::"r"(tmem + (uint32_t)(d * NS)), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                        }
                    }
                    if (CL == 1)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                                     ::"r"(smem_u32(&empty[st])) : "memory");
                    else                                 // the slot is free only when both CTAs consumed it
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                                     " [%0], %1;\n" ::"r"(smem_u32(&empty[st])), "h"((uint16_t)((1u << CL) - 1)) : "memory");
                    if ((c + 1) % FLUSH == 0 || c + 1 == nch)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                                     ::"r"(smem_u32(tfull)) : "memory");
                }
                __syncwarp();
                if ((c + 1) % FLUSH == 0 || c + 1 == nch) ++flush;
            }
        }
    } else if (warp < 4) {
        // ------------------------------------------------------------ epilogue (row = tid)
        uint32_t flush = 0;
        for (int64_t item = item0; item < nitems; item += istep) {
            const int i = nt - 1 - (int)(item / nbg), blk = (int)(item % nbg) * CL + crank;
            const int nch = 4 * (i + 1);
            double acc[NS];
#pragma unroll
            for (int j = 0; j < NS; ++j) acc[j] = 0.0;
            const int nflush = (nch + FLUSH - 1) / FLUSH;
            for (int f = 0; f < nflush; ++f, ++flush) {
                oz_mbar_wait(tfull, flush & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll 1
                for (int d = 0; d < S; ++d) {
                    const double sc = ldexp(1.0, -7 * (d + 2));
#pragma unroll
                    for (int cg = 0; cg < NS; cg += 16) {
                        uint32_t v[16];
                        const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(d * NS + cg);
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                                     : "r"(addr));
                        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc[cg + j] = fma((double)(int32_t)v[j], sc, acc[cg + j]);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;\n");
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty);
            }
            // first failing row per draw column: X_kj = acc_j 2^{e_k + 4} <= a_k
            const int64_t row = (int64_t)i * kTile + tid;
            const bool live = row < n;
            const double scale = live ? rowscale[row] * 16.0 : 0.0;
            const double ar = live ? a[row] : 0.0;
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                const bool fail = live && !(acc[j] * scale > ar);
                const unsigned m = __ballot_sync(0xffffffffu, fail);
                const int64_t s = (int64_t)blk * NS + j;
                if (m && lane == (j & 31) && s < ns) atomicMin(first + s, (int)(i * kTile + warp * 32 + __ffs(m) - 1));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (CL > 1) cluster_sync_all();             // no CTA leaves while its peer may still write into it
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(oz::TMEM_COLS));
}

// ------------------------------------------------------------------------------------------
// Level-split variant (method 2): the M128 N64 shape above runs the int8 tensor cores at half rate
// because 8 level accumulators x 64 columns fill the 512 TMEM columns. Here a 2-CTA cluster works
// on ONE item of 128 draws at the full-rate M128 N128 shape and splits the 36 products by level:
// CTA 0 owns levels {0, 1, 6, 7}, CTA 1 levels {2, 3, 4, 5} (18 products each, 4 accumulators x 128
// columns = 512 TMEM columns per CTA). CTA 0 multicasts the A (L-slice) chunk and CTA 1 the B
// (z-slice) chunk into both rings. At the end of an item each CTA owns one 64-draw half: 8 epilogue
// warps (TMEM lane quarter w % 4, column half w / 4) hand the half they do not own to the peer
// through an L2-resident scratch (double-buffered by item parity) and a remote mbarrier arrive,
// add the peer's contribution for their own half and take the first-failure decisions.
namespace oz2 {
constexpr int NS = 128;
constexpr int A_BYTES = oz::S * kTile * oz::KC;      // 32 KB
constexpr int B_SLICE = NS * oz::KC;                  // 4 KB
constexpr int B_BYTES = oz::S * B_SLICE;              // 32 KB
constexpr int STAGE = A_BYTES + B_BYTES;              // 64 KB
#ifndef MVN_OZ2_STAGES
#define MVN_OZ2_STAGES 3
#endif
constexpr int STAGES = MVN_OZ2_STAGES;           // (experiment knob: bytes in flight per CTA)
constexpr int NT = 320;                               // 8 epilogue warps + producer + MMA issuer
constexpr int SMEM = STAGES * STAGE + 1024;
}  // namespace oz2

constexpr uint32_t oz2_idesc() {   // kind::i8: D s32, A/B signed, K-major, N = 128, M = 128
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(oz2::NS >> 3) << 17) | ((uint32_t)(kTile >> 4) << 24);
}


__global__ void __launch_bounds__(oz2::NT, 1) k_oz2_trmm(const int8_t *__restrict__ LA, const int8_t *__restrict__ ZB,
                                                        int64_t n, int nt, int nblk, int64_t ns,
                                                        const double *__restrict__ rowscale, const double *__restrict__ a,
                                                        int *__restrict__ first, double *__restrict__ xch) {
    using namespace oz2;
    extern __shared__ __align__(1024) uint8_t smo[];
    uint8_t *ring = smo;
    uint64_t *full = reinterpret_cast<uint64_t *>(smo + STAGES * STAGE);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 1;
    uint64_t *xbar = tempty + 1;                        // peer's exchange data ready (4 warps arrive)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(xbar + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int crank = (int)cluster_rank();
    const int nchunk_all = nt * 4;
    const int64_t nitems = (int64_t)nt * nblk;
    const int64_t item0 = blockIdx.x / 2, istep = gridDim.x / 2;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 2); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);
        mbar_init(xbar, 4);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = *tmem_slot;
    // this CTA's four levels (global level d: products p + q = d + 2, 1-based)
    const int lv0 = crank == 0 ? 0 : 2, lv1 = crank == 0 ? 1 : 3, lv2 = crank == 0 ? 6 : 4, lv3 = crank == 0 ? 7 : 5;

    if (warp == 8) {
        // ------------------------------------------------------------ producer: my operand, to both CTAs
        if (lane == 0) {
            uint32_t q = 0;
            for (int64_t item = item0; item < nitems; item += istep) {
                const int i = nt - 1 - (int)(item / nblk), blk = (int)(item % nblk);
                const int nch = 4 * (i + 1);
                const int8_t *Ai = LA + 2ll * i * (i + 1) * A_BYTES;
                const int8_t *Bb = ZB + (int64_t)blk * nchunk_all * B_BYTES;
                for (int c = 0; c < nch; ++c, ++q) {
                    const int st = q % STAGES;
                    mbar_wait(&empty[st], ((q / STAGES) & 1) ^ 1);
                    uint8_t *dst = ring + st * STAGE;
                    mbar_arrive_expect_tx(&full[st], STAGE);
                    const uint8_t *src = crank == 0 ? (const uint8_t *)(Ai + (int64_t)c * A_BYTES)
                                                    : (const uint8_t *)(Bb + (int64_t)c * B_BYTES);
                    uint8_t *d = crank == 0 ? dst : dst + A_BYTES;
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                                 " [%0], [%1], %2, [%3], %4;\n"
                                 ::"r"(smem_u32(d)), "l"(src), "r"(A_BYTES), "r"(smem_u32(&full[st])), "h"((uint16_t)3) : "memory");
                }
            }
        }
    } else if (warp == 9) {
        // ------------------------------------------------------------ MMA issuer (18 products / chunk)
        uint32_t q = 0, flush = 0;
        constexpr uint32_t idesc = oz2_idesc();
        for (int64_t item = item0; item < nitems; item += istep) {
            const int i = nt - 1 - (int)(item / nblk);
            const int nch = 4 * (i + 1);
            for (int c = 0; c < nch; ++c, ++q) {
                const bool fresh = (c % oz::FLUSH) == 0;
                if (fresh) {
                    mbar_wait(tempty, (flush & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                }
                const int st = q % STAGES;
                mbar_wait(&full[st], (q / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(ring + st * STAGE), b0 = a0 + A_BYTES;
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        const int d = l == 0 ? lv0 : l == 1 ? lv1 : l == 2 ? lv2 : lv3;
                        for (int p = 0; p <= d; ++p) {
                            const uint64_t da = oz_desc(a0 + p * (kTile * oz::KC)), db = oz_desc(b0 + (d - p) * B_SLICE);
                            const uint32_t acc = (fresh && p == 0) ? 0u : 1u;
                            asm volatile("{\n .reg .pred pp;\n setp.ne.u32 pp, %4, 0;\n"
                                         " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp;\n}\n"
                                         ::"r"(tmem + (uint32_t)(l * NS)), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                        }
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                                 " [%0], %1;\n" ::"r"(smem_u32(&empty[st])), "h"((uint16_t)3) : "memory");
                    if ((c + 1) % oz::FLUSH == 0 || c + 1 == nch)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                                     ::"r"(smem_u32(tfull)) : "memory");
                }
                __syncwarp();
                if ((c + 1) % oz::FLUSH == 0 || c + 1 == nch) ++flush;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue: row = 32 (w%4) + lane, half h = w/4
        const int quarter = warp & 3, h = warp >> 2;
        const int row_in_tile = quarter * 32 + lane;
        const uint32_t peer_xbar = mapa_peer(smem_u32(xbar), (uint32_t)(crank ^ 1));
        uint32_t flush = 0, it = 0;
        for (int64_t item = item0; item < nitems; item += istep, ++it) {
            const int i = nt - 1 - (int)(item / nblk), blk = (int)(item % nblk);
            const int nch = 4 * (i + 1);
            double acc[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = 0.0;
            const int nflush = (nch + oz::FLUSH - 1) / oz::FLUSH;
            for (int f = 0; f < nflush; ++f, ++flush) {
                mbar_wait(tfull, flush & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
#pragma unroll 1
                for (int l = 0; l < 4; ++l) {
                    const int d = l == 0 ? lv0 : l == 1 ? lv1 : l == 2 ? lv2 : lv3;
                    const double sc = ldexp(1.0, -7 * (d + 2));
#pragma unroll
                    for (int cg = 0; cg < 64; cg += 16) {
                        uint32_t v[16];
                        const uint32_t addr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(l * NS + h * 64 + cg);
                        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                                     : "r"(addr));
                        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                        for (int j = 0; j < 16; ++j) acc[cg + j] = fma((double)(int32_t)v[j], sc, acc[cg + j]);
                    }
                }
                asm volatile("tcgen05.fence::before_thread_sync;\n");
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty);
            }
            // exchange: scratch [cluster][parity][half][128 rows][64] doubles
            double *X = xch + ((((int64_t)(blockIdx.x / 2) * 2 + (it & 1)) * 2 + h) * kTile + row_in_tile) * 64;
            if (h != crank) {
#pragma unroll
                for (int j = 0; j < 64; j += 2) *reinterpret_cast<double2 *>(X + j) = make_double2(acc[j], acc[j + 1]);
                __threadfence();
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(peer_xbar) : "memory");
                continue;
            }
            mbar_wait_cluster(xbar, it & 1);
#pragma unroll
            for (int j = 0; j < 64; j += 2) {
                const double2 v2 = __ldcg(reinterpret_cast<const double2 *>(X + j));
                acc[j] += v2.x;
                acc[j + 1] += v2.y;
            }
            const int64_t row = (int64_t)i * kTile + row_in_tile;
            const bool live = row < n;
            const double scale = live ? rowscale[row] * 16.0 : 0.0;
            const double ar = live ? a[row] : 0.0;
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const bool fail = live && !(acc[j] * scale > ar);
                const unsigned m = __ballot_sync(0xffffffffu, fail);
                const int64_t s = (int64_t)blk * NS + h * 64 + j;
                if (m && lane == (j & 31) && s < ns) atomicMin(first + s, (int)(row - lane + __ffs(m) - 1));
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
}

cudaError_t mc_oz_init() {
    cudaError_t e = cudaFuncSetAttribute(k_oz_trmm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, oz::SMEM);
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_oz2_trmm, cudaFuncAttributeMaxDynamicSharedMemorySize, oz2::SMEM))) return e;
    return cudaFuncSetAttribute(k_oz_trmm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, oz::SMEM);
}

// Cluster size of k_oz_trmm (MVN_MC_CLUSTER: 1 or 2). Measured at D (r01): 53.35 (1) vs 53.25 (2)
// fp64-equivalent TFLOP/s — the shared-operand traffic is not the limiter; the MMA shape is:
// tcgen05 kind::i8 runs M128 N64 (and M64 N128) at half the M128 N128 rate (3,890 vs 7,381
// MAC/clk/SM, tools/umma_i8_test.cu, tools/umma_i8_m64.cu), and 8 level accumulators of 128
// columns do not fit the 512 TMEM columns. Default 1.
int mc_oz_cluster() {
    static const int v = [] { const char *e = getenv("MVN_MC_CLUSTER"); const int x = e ? atoi(e) : 1; return x == 2 ? 2 : 1; }();
    return v;
}

int64_t mc_oz_la_bytes(int64_t n) {
    const int64_t nt = (n + kTile - 1) / kTile;
    return 2 * nt * (nt + 1) * oz::A_BYTES;
}
int64_t mc_oz_zb_bytes(int64_t n, int64_t ns) {        // draw blocks rounded up to a multiple of 2
    const int64_t nt = (n + kTile - 1) / kTile;
    const int64_t nblk = ((ns + oz::NS - 1) / oz::NS + 1) / 2 * 2;
    return nblk * nt * 4 * oz::B_BYTES;
}

cudaError_t launch_mc_oz_prepare(int64_t n, const double *tiles, double *rowscale, int8_t *LA, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int64_t rows = (int64_t)nt * kTile;
    k_oz_rowscale<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(tiles, n, nt, rowscale);
    const int64_t threads = 2ll * nt * (nt + 1) * kTile;
    k_oz_lslice<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(tiles, nt, rowscale, LA);
    return cudaGetLastError();
}

cudaError_t launch_mc_oz_chunk(int64_t n, const int8_t *LA, const double *rowscale, const double *a, uint64_t seed,
                               int64_t s0, int64_t ns, int8_t *ZB, int *first, unsigned long long *count, int nsm,
                               cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int CL = mc_oz_cluster();
    const int nblk = (int)(((ns + oz::NS - 1) / oz::NS + CL - 1) / CL * CL);   // padded draws are zero
    const int64_t total = (int64_t)nblk * nt * 4 * oz::KC * oz::NS;
    k_oz_zgen<oz::NS><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(ZB, n, nt * 4, s0, ns, seed, total);
    cudaError_t e = launch_mc_first_init(first, ns, (int)n, st);
    if (e != cudaSuccess) return e;
    const int64_t items = (int64_t)nt * (nblk / CL);
    const int grid = (int)std::min<int64_t>(items, nsm / CL) * CL;
    if (CL == 1) {
        k_oz_trmm<1><<<grid, oz::NT, oz::SMEM, st>>>(LA, ZB, n, nt, nblk, ns, rowscale, a, first);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        // co-resident clusters of 2 (a GPC with an odd SM count leaves one SM out): persistent grid
        static int max_clusters = 0;
        if (!max_clusters) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(2);
            q.blockDim = dim3(oz::NT);
            q.dynamicSmemBytes = oz::SMEM;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = 2; qa[0].val.clusterDim.y = 1; qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&max_clusters, k_oz_trmm<2>, &q) != cudaSuccess || max_clusters < 1)
                max_clusters = nsm / 2;
        }
        cfg.gridDim = dim3((unsigned)(std::min<int64_t>(items, max_clusters) * 2));
        cfg.blockDim = dim3(oz::NT);
        cfg.dynamicSmemBytes = oz::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e2 = cudaLaunchKernelEx(&cfg, k_oz_trmm<2>, LA, ZB, n, nt, nblk, ns, rowscale, a, first);
        if (e2 != cudaSuccess) return e2;
    }
    return launch_mc_count(first, ns, count, st);
}


int64_t mc_oz2_zb_bytes(int64_t n, int64_t ns) {
    const int64_t nt = (n + kTile - 1) / kTile;
    return (ns + oz2::NS - 1) / oz2::NS * nt * 4 * oz2::B_BYTES;
}
int64_t mc_oz2_xch_bytes(int nsm) { return (int64_t)(nsm / 2) * 2 * 2 * kTile * 64 * 8; }

cudaError_t launch_mc_oz2_chunk(int64_t n, const int8_t *LA, const double *rowscale, const double *a, uint64_t seed,
                                int64_t s0, int64_t ns, int8_t *ZB, double *xch, int *first, unsigned long long *count,
                                int nsm, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int nblk = (int)((ns + oz2::NS - 1) / oz2::NS);
    const int64_t total = (int64_t)nblk * nt * 4 * oz::KC * oz2::NS;
    k_oz_zgen<oz2::NS><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(ZB, n, nt * 4, s0, ns, seed, total);
    cudaError_t e = launch_mc_first_init(first, ns, (int)n, st);
    if (e != cudaSuccess) return e;
    const int64_t items = (int64_t)nt * nblk;
    static int max_clusters = 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(oz2::NT);
    cfg.dynamicSmemBytes = oz2::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (!max_clusters) {
        cfg.gridDim = dim3(2);
        if (cudaOccupancyMaxActiveClusters(&max_clusters, k_oz2_trmm, &cfg) != cudaSuccess || max_clusters < 1)
            max_clusters = nsm / 2;
        max_clusters = std::min(max_clusters, nsm / 2);    // the exchange scratch is sized for nsm / 2
    }
    cfg.gridDim = dim3((unsigned)(std::min<int64_t>(items, max_clusters) * 2));
    if ((e = cudaLaunchKernelEx(&cfg, k_oz2_trmm, LA, ZB, n, nt, nblk, ns, rowscale, a, first, xch))) return e;
    return launch_mc_count(first, ns, count, st);
}
}  // namespace mvn
