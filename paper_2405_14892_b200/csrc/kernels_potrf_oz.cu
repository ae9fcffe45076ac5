// NEXT-4 ("mixed precision ... tensor core execution") for the
// Cholesky (a3): the trailing update A_ij -= sum_{c in super-panel} L_ic L_jc^T (Alg. 1 l.8, P:233;
// box (a) of P:319) on the int8 tensor cores, an Ozaki-style split (reading R25): per
// super-step the panel's rows get a power-of-two scale over the panel's columns and 8 signed 7-bit
// digits (as the MC and SOV emulations), and each trailing tile is
//   A_ij -= 2^{e_i + e_j} sum_{d=0}^{7} 2^{-7(d+2)} sum_{p+q=d+2} (A_p(i) A_q(j)^T)     (36 int8 GEMMs)
// with K = 128 kp <= 1,024 per update, so every level sum is exact in int32 without a flush.
// Dropped terms: ~2^-53 2^{e_i+e_j} per update with random signs — the rounding of an fp64 GEMM.
// The panel factorisation (POTRF / TRSM / the look-ahead update) stays on fp64 DMMA.
//
// Kernel (k_upd_oz): MC method 2's engine — a 2-CTA cluster per 128 x 128 tile, the 36 products
// split by level (CTA 0 {0, 1, 6, 7}, CTA 1 {2, 3, 4, 5}), M128 N128 K32 MMAs into 4 x 128 TMEM
// columns, CTA 0 multicasting the A chunk (rows of tile i), CTA 1 the B chunk (rows of tile j) into
// a 3-stage ring; 8 epilogue warps drain TMEM, swap the column half they do not own with the peer
// through an L2 scratch, and subtract the scaled result from the tile in place.
#include <algorithm>

#include "common.cuh"
#include "mvn_internal.h"
#include "umma.cuh"

namespace mvn {
namespace poz {
constexpr int KC = 32;
constexpr int NSL = 8;
constexpr int SLICE = kTile * KC;   // 4 KB
constexpr int HALF = NSL * SLICE;   // 32 KB: the 8 slices of one 128-row x 32-column chunk
constexpr int STAGE = 2 * HALF;
constexpr int STAGES = 3;
constexpr int NT = 320;             // warps 0-7 epilogue, 8 producer, 9 MMA issuer
constexpr int SMEM = STAGES * STAGE + 1024;
}  // namespace poz

// Per-row power-of-two scale over the super-panel's columns k*128 .. (k+w)*128 - 1 for the rows of
// the trailing tiles (tile rows >= k + w): rs[r] = 2^{e+1} with max |L| < 2^e (so |L / rs| < 1/2).
__global__ void k_pan_rowscale(const double *__restrict__ tiles, int k, int w, int nt, double *__restrict__ rs) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r0 = (int64_t)(k + w) * kTile;
    if (r >= (int64_t)nt * kTile - r0) return;
    const int64_t gr = r0 + r;
    const int I = (int)(gr / kTile), rr = (int)(gr % kTile);
    double m = 0.0;
    for (int J = k; J < k + w; ++J) {
        const double *T = tiles + tile_offset(I, J) + rr;
        for (int c = 0; c < kTile; ++c) m = fmax(m, fabs(T[(int64_t)c * kTile]));
    }
    int e;
    frexp(m, &e);
    rs[r] = m > 0.0 ? ldexp(1.0, e + 1) : 1.0;
}

// The 8 digit slices of the panel rows in the tcgen05 K-major operand layout:
//   LAp[((I - (k+w)) * 4w + c) * HALF + p * SLICE + core(rr, kk)] = a_p(row, 32 c + kk)
// One thread per (row, 16 consecutive panel columns): 16 digits per slice = one 16-byte store;
// consecutive threads take consecutive rows (coalesced column reads of the column-major tiles).
__global__ void k_pan_slice(const double *__restrict__ tiles, int k, int w, int nt, const double *__restrict__ rs,
                            int8_t *__restrict__ LAp) {
    using namespace poz;
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t ntr = nt - k - w;                       // trailing tile rows
    const int groups = 8 * w;                             // 16-column groups of the panel
    if (gid >= ntr * groups * kTile) return;
    const int rr = (int)(gid % kTile);
    const int64_t t = gid / kTile;
    const int g = (int)(t % groups);
    const int64_t Ip = t / groups;                        // trailing tile row, 0-based
    const int c = g >> 1, kh = g & 1;                     // 32-column chunk, 16-column half
    const int J = k + (c >> 2), col0 = (c & 3) * KC + kh * 16;
    const int64_t I = k + w + Ip;
    const double *T = tiles + tile_offset(I, J) + rr;
    const double inv = 1.0 / rs[Ip * kTile + rr];         // exact: a power of two
    uint32_t dg[NSL][4];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        double v = T[(int64_t)(col0 + q) * kTile] * inv;
#pragma unroll
        for (int p = 0; p < NSL; ++p) {
            v *= 128.0;
            const double d = rint(v);
            v -= d;
            const uint32_t b = (uint32_t)((int)d & 0xff) << ((q & 3) * 8);
            if ((q & 3) == 0) dg[p][q >> 2] = b; else dg[p][q >> 2] |= b;
        }
    }
    int8_t *dst = LAp + (Ip * 4 * w + c) * (int64_t)HALF + ((rr >> 3) << 8) + (kh << 7) + ((rr & 7) << 4);
#pragma unroll
    for (int p = 0; p < NSL; ++p)
        *reinterpret_cast<uint4 *>(dst + p * SLICE) = make_uint4(dg[p][0], dg[p][1], dg[p][2], dg[p][3]);
}

struct UpdOzArgs {
    double *tiles;
    const int8_t *LAp;
    const double *rs;
    double *xch;              // [clusters][2 parity][2 halves][128][64]
    int k, w, nt, c0, cs, cb;
    int64_t nitems;
};

__device__ __forceinline__ int poz_level(int crank, int l) { return crank == 0 ? (l < 2 ? l : l + 4) : l + 2; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(poz::NT, 1) k_upd_oz(const UpdOzArgs p) {
    using namespace poz;
    extern __shared__ __align__(1024) uint8_t smo[];
    uint8_t *ring = smo;
    uint64_t *full = reinterpret_cast<uint64_t *>(smo + STAGES * STAGE);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES, *tempty = tfull + 1, *xbar = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfull + 3);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int crank = (int)cluster_rank();
    const int64_t item0 = blockIdx.x >> 1, istep = gridDim.x >> 1;
    const int nch = 4 * p.w;
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

    if (warp == 8) {
        // ------------------------------------------------------------ producer: my operand, to both CTAs
        if (lane == 0) {
            uint32_t q = 0;
            int64_t base = 0;
            int col = 0;
            for (int64_t item = item0; item < p.nitems; item += istep) {
                int ti, tj;
                upd_item(item, p.nt, p.c0, p.cs, p.cb, ti, tj, base, col);
                const int Ip = (crank == 0 ? ti : tj) - p.k - p.w;
                const int8_t *src0 = p.LAp + (int64_t)Ip * nch * HALF;
                for (int c = 0; c < nch; ++c, ++q) {
                    const int st = q % STAGES;
                    mbar_wait(&empty[st], ((q / STAGES) & 1) ^ 1);
                    uint8_t *dst = ring + st * STAGE + (crank == 0 ? 0 : HALF);
                    mbar_arrive_expect_tx(&full[st], STAGE);
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                                 " [%0], [%1], %2, [%3], %4;\n"
                                 ::"r"(smem_u32(dst)), "l"(src0 + (int64_t)c * HALF), "r"(HALF), "r"(smem_u32(&full[st])),
                                   "h"((uint16_t)3) : "memory");
                }
            }
        }
    } else if (warp == 9) {
        // ------------------------------------------------------------ MMA issuer (18 products per chunk)
        uint32_t q = 0, it = 0;
        constexpr uint32_t idesc = i8_idesc(kTile);
        for (int64_t item = item0; item < p.nitems; item += istep, ++it) {
            for (int c = 0; c < nch; ++c, ++q) {
                if (c == 0) {
                    mbar_wait(tempty, (it & 1) ^ 1);          // the previous tile drained
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                }
                const int st = q % STAGES;
                mbar_wait(&full[st], (q / STAGES) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(ring + st * STAGE), b0 = a0 + HALF;
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        const int d = poz_level(crank, l);
                        for (int pp = 0; pp <= d; ++pp) {
                            const uint64_t da = oz_desc(a0 + pp * SLICE), db = oz_desc(b0 + (d - pp) * SLICE);
                            const uint32_t acc = (c == 0 && pp == 0) ? 0u : 1u;
                            asm volatile("{\n .reg .pred pp;\n setp.ne.u32 pp, %4, 0;\n"
                                         " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp;\n}\n"
                                         ::"r"(tmem + (uint32_t)(l * kTile)), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                        }
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                                 " [%0], %1;\n" ::"r"(smem_u32(&empty[st])), "h"((uint16_t)3) : "memory");
                    if (c + 1 == nch)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                                     ::"r"(smem_u32(tfull)) : "memory");
                }
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue: row = 32 (w % 4) + lane, column half w / 4
        const int quarter = warp & 3, h = warp >> 2;
        const int row = quarter * 32 + lane;
        const uint32_t peer_xbar = mapa_peer(smem_u32(xbar), (uint32_t)(crank ^ 1));
        uint32_t it = 0;
        int64_t base = 0;
        int col = 0;
        for (int64_t item = item0; item < p.nitems; item += istep, ++it) {
            int ti, tj;
            upd_item(item, p.nt, p.c0, p.cs, p.cb, ti, tj, base, col);
            double acc[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = 0.0;
            mbar_wait(tfull, it & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n");
            // per 16-column group: the 4 levels' loads in flight together, one wait
#pragma unroll
            for (int cg = 0; cg < 64; cg += 16) {
                uint32_t v[4][16];
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const uint32_t addr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(l * kTile + h * 64 + cg);
                    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                                 : "=r"(v[l][0]), "=r"(v[l][1]), "=r"(v[l][2]), "=r"(v[l][3]), "=r"(v[l][4]), "=r"(v[l][5]),
                                   "=r"(v[l][6]), "=r"(v[l][7]), "=r"(v[l][8]), "=r"(v[l][9]), "=r"(v[l][10]), "=r"(v[l][11]),
                                   "=r"(v[l][12]), "=r"(v[l][13]), "=r"(v[l][14]), "=r"(v[l][15])
                                 : "r"(addr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const double sc = ldexp(1.0, -7 * (poz_level(crank, l) + 2));
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc[cg + j] = fma((double)(int32_t)v[l][j], sc, acc[cg + j]);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n");
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
            // exchange through L2: [cluster][parity][half][128 rows][64]
            double *X = p.xch + ((((int64_t)(blockIdx.x >> 1) * 2 + (it & 1)) * 2 + h) * kTile + row) * 64;
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
            // A_ij[row][h*64 + j] -= (acc + peer) * 2^{e_row} * 2^{e_col}
            const double sr = p.rs[(int64_t)(ti - p.k - p.w) * kTile + row];
            const double *rsj = p.rs + (int64_t)(tj - p.k - p.w) * kTile + h * 64;
            double *C = p.tiles + tile_offset(ti, tj) + (int64_t)(h * 64) * kTile + row;
            // in batches of 16 columns: all loads of a batch in flight before the first use (the
            // epilogue must finish before this warp can drain the next tile's accumulators)
#pragma unroll
            for (int jb = 0; jb < 64; jb += 16) {
                double cv[16], xv[16], rv[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    cv[j] = C[(int64_t)(jb + j) * kTile];
                    xv[j] = __ldcg(X + jb + j);
                    rv[j] = __ldg(rsj + jb + j);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) C[(int64_t)(jb + j) * kTile] = cv[j] - (acc[jb + j] + xv[j]) * sr * rv[j];
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
}

cudaError_t potrf_oz_init() {
    return cudaFuncSetAttribute(k_upd_oz, cudaFuncAttributeMaxDynamicSharedMemorySize, poz::SMEM);
}

int potrf_oz_max_clusters(int nsm) {
    static int cached = 0;
    if (!cached) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(poz::NT);
        cfg.dynamicSmemBytes = poz::SMEM;
        int v = 0;
        if (cudaOccupancyMaxActiveClusters(&v, k_upd_oz, &cfg) != cudaSuccess || v < 1) {
            cudaGetLastError();
            v = nsm / 2;
        }
        cached = std::min(v, nsm / 2);
    }
    return cached;
}

int64_t potrf_oz_lap_bytes(int64_t n, int kp) {
    const int64_t nt = (n + kTile - 1) / kTile;
    return std::max<int64_t>(nt - 1, 1) * 4 * kp * poz::HALF;
}
int64_t potrf_oz_xch_bytes(int clusters) { return (int64_t)clusters * 4 * kTile * 64 * 8; }

// A_ij -= sum_{c=k}^{k+w-1} L_ic L_jc^T on the int8 tensor cores for the tile columns of the filter
// (c0, cs, cb) (all >= k + w), on `clusters` 2-CTA clusters: slice the panel, then the update.
cudaError_t launch_potrf_update_oz(int64_t n, double *tiles, int k, int w, int c0, int cs, int cb, int clusters,
                                   int8_t *LAp, double *rs, double *xch, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    if (c0 >= nt) return cudaSuccess;
    w = std::min(w, nt - k);
    const int64_t rows = (int64_t)(nt - k - w) * kTile;
    if (rows <= 0) return cudaSuccess;
    k_pan_rowscale<<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(tiles, k, w, nt, rs);
    const int64_t thr = rows * 8 * w;
    k_pan_slice<<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(tiles, k, w, nt, rs, LAp);
    UpdOzArgs a;
    a.tiles = tiles; a.LAp = LAp; a.rs = rs; a.xch = xch; a.k = k; a.w = w; a.nt = nt; a.c0 = c0; a.cs = cs; a.cb = cb;
    a.nitems = upd_items(nt, c0, cs, cb);
    const int cl = (int)std::min<int64_t>(clusters, a.nitems);
    k_upd_oz<<<2 * cl, poz::NT, poz::SMEM, st>>>(a);
    return cudaGetLastError();
}

}  // namespace mvn
