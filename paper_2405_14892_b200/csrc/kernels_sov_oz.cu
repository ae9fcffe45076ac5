// NEXT-4 ("mixed precision ... tensor core execution", the paper's stated
// future work) for the SOV sweep (a6-a8): the GEMM update S = L Y of Alg. 2 l.10-13
// on the int8 tensor cores (tcgen05.mma kind::i8, int32 accumulators in TMEM), exact int8 products
// combined in fp64 — an Ozaki-style split (reading R24) — while the Phi / Phi^{-1} chain
// (Alg. 3, a7), the in-block part of s and the per-prefix log-sum-exp (a8) stay in fp64 exactly as in
// k_sov. Opt-in (mvn_sov_prefix_ex, method 1); the fp64 DMMA sweep stays the default.
//
//   L_kt = 2^{e_k} sum_{p=1..8} a_p(k,t) 2^{-7p},  |L_kt| < 2^{e_k - 1}   (per-row exponent, k_oz_lslice)
//   y    = 2^7     sum_{q=1..8} b_q       2^{-7q},  |y| < 63.5           (fixed exponent)
//   s_k  = 2^{e_k + 7} sum_{d=0}^{7} 2^{-7(d+2)} sum_{p+q=d+2} (A_p B_q)      (36 int8 GEMMs, 8 levels)
// Every level sum is exact in int32 (|level| <= 8 * 64 * 64 * K < 2^31 for K <= 32,768 per flush).
// Dropped: the pairs p + q > 9 and the digits beyond the 8th, ~2^-47 of 2^{e_k+7} per K-term with
// random signs (absolute error of s ~1e-13 at K = 65,536), far inside the north_star's 1e-8 on log P.
//
// Full-rate layout (the MC kernel's method 2, profiles/r01_umma_i8_2sm.txt, r02_mc2_ring_depth.md):
// a CLUSTER OF 2 CTAs sweeps one block of 128 samples; the MMA is D[128 samples][128 rows] (M = the
// samples on the TMEM lanes, N = the 128 rows of one tile row, K = 32 per chunk), split by level —
// CTA 0 keeps levels {0, 1, 6, 7}, CTA 1 levels {2, 3, 4, 5}: 18 MMAs per chunk and 4 x 128 TMEM
// columns (all 512) each. CTA 0 multicasts the L-slice chunk, CTA 1 the Y-slice chunk into both
// CTAs' 2-stage rings. The chain of CTA c runs samples 64c .. 64c+63 (TMEM lanes of warps 2c, 2c+1);
// the other two lane quarters hold the peer's samples: those warps convert their levels to fp64
// and hand them over through an L2 scratch (remote mbarrier arrive), so each chain sees all 8 levels.
//
// Per CTA, 6 warps:
//   warps 0-3 : TMEM lane quarters; quarter q belongs to CTA q / 2's chain: "chain" warps run Alg. 3 on
//               their samples (S from TMEM + the peer's part, in-block dots from the diagonal tile in
//               fp64, y -> 8 int8 digits -> the cluster's Y-slice history in HBM), "exchange" warps
//               drain the peer's samples;
//   warp 4    : producer (one lane): two bulk copies per chunk, multicast;
//   warp 5    : MMA issuer (one lane).
// Row block rb (128 rows) needs Y of rows < 128 rb: the MMA of rb + 1 runs while the chain does rb,
// and only the chunks of row block rb wait for its Y (barrier yready in CTA 1, one arrive per CTA).
#include <algorithm>

#include "common.cuh"
#include "mvn_internal.h"
#include "normal.cuh"
#include "umma.cuh"

namespace mvn {
namespace soz {
constexpr int NSB = 128;            // samples per block (MMA M = TMEM lanes)
constexpr int RB = 128;             // rows per row block (MMA N) = one tile row
constexpr int KC = 32;              // K per chunk (one kind::i8 MMA)
constexpr int NSL = 8;              // slices per operand
constexpr int SLICE = 128 * KC;     // 4 KB: [128 rows x 32 K] int8 in core-matrix order
constexpr int HALF = NSL * SLICE;   // 32 KB: all slices of one operand chunk
constexpr int STAGE = 2 * HALF;     // 64 KB: A (Y^T slices) + B (L slices)
constexpr int STAGES = 2;
constexpr int FLUSH = 1024;         // chunks per TMEM flush (K = 32,768: level sums < 2^31)
constexpr int CS = 64;              // samples of one CTA's chain
constexpr int NT = 192;
constexpr int OFF_S = STAGES * STAGE;                 // double S[128 rows][64]
constexpr int OFF_PAN = OFF_S + RB * CS * 8;          // double panel[2][8 cols][128 rows]
constexpr int OFF_PS = OFF_PAN + 2 * 8 * RB * 8;      // double ps[128 rows][2 warps][2]
constexpr int OFF_E8 = OFF_PS + RB * 2 * 2 * 8;       // double ELL8[8][64], P8[8][64]
constexpr int OFF_AG = OFF_E8 + 2 * 8 * CS * 8;       // double a[128], G[128] (bits), dinv[128], scale[128]
constexpr int OFF_BAR = OFF_AG + 4 * RB * 8;
constexpr int SMEM = OFF_BAR + 128;
enum : int { BAR_CH = 1, BAR_EX = 2 };                // named barriers: chain warps, exchange warps (64 each)
}  // namespace soz

struct SovOzArgs {
    const int8_t *LA;         // L slices: row tile i, chunk c at (2 i (i+1) + c) * HALF (k_oz_lslice)
    const double *rowscale;   // 2^{e_k}
    const double *L;          // fp64 tiles (the diagonal tiles: in-block part, 1 / L_kk)
    int64_t n, n_pad;         // n_pad = nrb * 128
    int nrb;
    const double *a;          // lower limits (b = +inf)
    const uint64_t *G;
    int64_t N;
    uint64_t seed;
    const int64_t *cl;        // [clusters][3]: first global sample, count, first block index
    int8_t *YS;               // [clusters][nrb * 4 chunks][HALF]: the Y-slice history
    double *xch;              // [clusters][2 destination CTA][2 parity][128 rows][64]
    double *part;             // [2 * blocks][n_pad][2]: (max ell, sum e^{ell - max}) per CTA half-block
    int *flag;                // set when |y| >= 63.5 (outside the fixed y scale)
    // soft cluster lockstep (L2 reuse of the shared L-slice stream; 0 = off): CTA 0's producer starts
    // step t = b (nrb - 1) + rb - 1 only when every cluster that has step t - lag has issued it
    int lag;
    int *step_done;           // [max blocks * (nrb - 1)] issue counters (zeroed per launch)
    const int *need;          // [max blocks]: clusters with more than b blocks
};

__device__ __forceinline__ uint64_t soz_shift(uint64_t seed, uint64_t r, uint64_t k) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * ((r << 32) + k + 1ull);   // reading R8
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double soz_w(uint64_t j, uint64_t G, uint64_t D) {
    return ((double)((j * G + D) >> 12) + 0.5) * 0x1p-52;
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(addr));
}

// This CTA's four levels d (products p + q = d + 2, 1-based slices).
__device__ __forceinline__ int soz_level(int crank, int l) {
    return crank == 0 ? (l < 2 ? l : l + 4) : l + 2;
}

// Drain one flush of this warp's TMEM lane quarter: for the 128 rows, P = sum_l 2^{-7(d_l+2)} D_l
// (exact int32 -> fp64, power-of-two scales), written (first flush) or added to dst[row * 64 + jj].
__device__ __forceinline__ void soz_drain(uint32_t tmem, int quarter, int crank, double *dst, int jj, bool first) {
#pragma unroll 1
    for (int cg = 0; cg < soz::RB; cg += 16) {
        double P[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) P[i] = 0.0;
        uint32_t v[4][16];                                 // the 4 levels' loads in flight together
#pragma unroll
        for (int l = 0; l < 4; ++l) tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(l * soz::RB + cg), v[l]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const double sc = ldexp(1.0, -7 * (soz_level(crank, l) + 2));
#pragma unroll
            for (int i = 0; i < 16; ++i) P[i] = fma((double)(int32_t)v[l][i], sc, P[i]);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            double *q = dst + (cg + i) * soz::CS + jj;
            *q = first ? P[i] : *q + P[i];
        }
    }
}

// Alg. 3 on one row block of 128 rows for sample jj (local) of this CTA's chain: k_sov's
// chain_rowblock with 64 samples and 128-row blocks. s of row li arrives in S[li][jj] (GEMM part,
// scaled, + in-block contributions so far); the diagonal tile comes through 8-column panels.
// y goes to S (in-block updates of the later rows) and, as 8 int8 digits, to the Y-slice history.
__device__ __forceinline__ void soz_chain_rowblock(const SovOzArgs &p, uint8_t *smo, int rb, int jj, int m, bool valid,
                                                   uint64_t r, uint64_t jl, double &ell, int8_t *YS, int tid_ch) {
    using namespace soz;
    double *S = reinterpret_cast<double *>(smo + OFF_S);
    double *pan = reinterpret_cast<double *>(smo + OFF_PAN);
    double *ps = reinterpret_cast<double *>(smo + OFF_PS);
    double *ELL8 = reinterpret_cast<double *>(smo + OFF_E8), *P8 = ELL8 + 8 * CS;
    const double *a_s = reinterpret_cast<const double *>(smo + OFF_AG);
    const uint64_t *G_s = reinterpret_cast<const uint64_t *>(a_s + RB);
    const double *dinv = a_s + 2 * RB;
    const int64_t row0 = (int64_t)rb * RB;
    const double *Dt = p.L + tile_offset(rb, rb);            // column-major diagonal tile
    const int lane = jj & 31, cw = jj >> 5;
    uint64_t dlo[NSL], dhi[NSL];                              // 16 rows x 8 digits: bytes 0-7, 8-15
    bool big = false;
    // panel 0 of this row block
    {
        const double *src = Dt;
#pragma unroll
        for (int e = 0; e < 8; ++e) cp_async16(pan + (e * 64 + tid_ch) * 2, src + (e * 64 + tid_ch) * 2);
        cp_async_commit();
    }
#pragma unroll 1
    for (int sb = 0; sb < RB / 8; ++sb) {
        const int rb0 = sb * 8;
        const int64_t left = p.n - (row0 + rb0);
        if (left <= 0) break;                                 // uniform
        const int nrows = left < 8 ? (int)left : 8;
        if (sb + 1 < RB / 8 && left > 8) {                    // next panel (columns rb0+8 .. rb0+15)
            const double *src = Dt + (int64_t)(rb0 + 8) * kTile;
            double *dst = pan + ((sb + 1) & 1) * 8 * RB;
#pragma unroll
            for (int e = 0; e < 8; ++e) cp_async16(dst + (e * 64 + tid_ch) * 2, src + (e * 64 + tid_ch) * 2);
        }
        cp_async_commit();
        cp_async_wait<1>();
        named_sync(BAR_CH, 64);                              // panel sb landed for both chain warps
        const double *Ld = pan + (sb & 1) * 8 * RB;           // Ld[c * 128 + row], c = column - rb0
        double s = S[rb0 * CS + jj];
        double c_w = valid ? ell : -CUDART_INF;
#pragma unroll
        for (int o = 16; o; o >>= 1) c_w = fmax(c_w, __shfl_xor_sync(0xffffffffu, c_w, o));
        double pw = (valid && c_w != -CUDART_INF) ? exp(ell - c_w) : 0.0;
#pragma unroll 1
        for (int i = 0; i < nrows; ++i) {
            const int li = rb0 + i;
            const int64_t k = row0 + li;
            const double s_next = (i + 1 < 8) ? S[(li + 1) * CS + jj] : 0.0;
            const double ap = (a_s[li] - s) * dinv[li];
            const double wq = soz_w(jl, G_s[li], soz_shift(p.seed, r, (uint64_t)k));
            double lq, y, q;
            sov_step_upper(ap, wq, lq, y, q);
            pw *= q;
            P8[i * CS + jj] = pw;
            ell += lq;
            S[li * CS + jj] = y;
            ELL8[i * CS + jj] = ell;
            if (i + 1 < 8) s = s_next + Ld[i * RB + li + 1] * y;
#pragma unroll
            for (int d = 2; d < 8; ++d)
                if (i + d < 8) S[(li + d) * CS + jj] += Ld[i * RB + li + d] * y;
        }
        // per-row log-sum-exp over this warp's 32 samples, 8 rows at once (k_sov's fast path)
        double mx[8], ex[8];
        double pmax = valid ? pw : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
        if (pmax >= 0x1p-960) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                mx[i] = c_w;
                ex[i] = (valid && i < nrows && c_w != -CUDART_INF) ? P8[i * CS + jj] : 0.0;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) mx[i] = (valid && i < nrows) ? ELL8[i * CS + jj] : -CUDART_INF;
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int i = 0; i < 8; ++i) mx[i] = fmax(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
#pragma unroll
            for (int i = 0; i < 8; ++i) ex[i] = (valid && i < nrows && mx[i] != -CUDART_INF) ? exp(ELL8[i * CS + jj] - mx[i]) : 0.0;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int i = 0; i < 8; ++i) ex[i] += __shfl_xor_sync(0xffffffffu, ex[i], o);
        if (lane < nrows) {
            double mi = mx[0], ei = ex[0];
#pragma unroll
            for (int i = 1; i < 8; ++i)
                if (lane == i) { mi = mx[i]; ei = ex[i]; }
            *reinterpret_cast<double2 *>(ps + ((rb0 + lane) * 2 + cw) * 2) = make_double2(mi, ei);
        }
        double yv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) yv[i] = S[(rb0 + i) * CS + jj];
        // the sub-block's y -> 8 digits each of y / 128 (reading R24: exact rint of the scaled
        // residual), off the row recursion's critical path: 8 independent y at a time; a 16-row group
        // of the Y-digit history (two sub-blocks) is stored as one 16-byte word per slice
        {
            uint64_t half[NSL];
#pragma unroll
            for (int qd = 0; qd < NSL; ++qd) half[qd] = 0ull;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double y = i < nrows ? yv[i] : 0.0;
                big |= !(fabs(y) < 63.5);
                double v = y * 0x1p-7;
#pragma unroll
                for (int qd = 0; qd < NSL; ++qd) {
                    v *= 128.0;
                    const double t = rint(v);
                    v -= t;
                    half[qd] |= (uint64_t)((uint32_t)(int)t & 0xffu) << (8 * i);
                }
            }
            if ((sb & 1) == 0) {
#pragma unroll
                for (int qd = 0; qd < NSL; ++qd) { dlo[qd] = half[qd]; dhi[qd] = 0ull; }
            } else {
#pragma unroll
                for (int qd = 0; qd < NSL; ++qd) dhi[qd] = half[qd];
            }
            if ((sb & 1) == 1 || left <= 8) {
                const int64_t k0 = row0 + (rb0 & ~15);          // first row of the 16-row group
                const int kk = (int)(k0 & 31);
                int8_t *dst = YS + (k0 >> 5) * (int64_t)HALF + ((m >> 3) << 8) + ((kk >> 4) << 7) + ((m & 7) << 4);
#pragma unroll
                for (int qd = 0; qd < NSL; ++qd)
                    *reinterpret_cast<uint4 *>(dst + qd * SLICE) =
                        make_uint4((uint32_t)dlo[qd], (uint32_t)(dlo[qd] >> 32), (uint32_t)dhi[qd], (uint32_t)(dhi[qd] >> 32));
            }
        }
#pragma unroll 2
        for (int li = rb0 + 8; li < RB; ++li) {
            double t = S[li * CS + jj];
#pragma unroll
            for (int i = 0; i < 8; ++i) t += Ld[i * RB + li] * yv[i];
            S[li * CS + jj] = t;
        }
        named_sync(BAR_CH, 64);                               // panel sb free for the prefetch of sb + 2
    }
    cp_async_wait<0>();
    if (big) atomicOr(p.flag, 1);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(soz::NT, 1) k_sov_oz(const SovOzArgs p) {
    using namespace soz;
    extern __shared__ __align__(1024) uint8_t smo[];
    uint8_t *ring = smo;
    double *Ssm = reinterpret_cast<double *>(smo + OFF_S);
    double *ps = reinterpret_cast<double *>(smo + OFF_PS);
    double *a_s = reinterpret_cast<double *>(smo + OFF_AG);
    uint64_t *G_s = reinterpret_cast<uint64_t *>(a_s + RB);
    double *dinv = a_s + 2 * RB, *scl = a_s + 3 * RB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smo + OFF_BAR);
    uint64_t *full = bars, *empty = bars + STAGES, *tfull = bars + 2 * STAGES, *tempty = tfull + 1, *xbar = tfull + 2,
             *yready = tfull + 3;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfull + 4);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int crank = (int)cluster_rank();
    const int clu = blockIdx.x >> 1;
    const int64_t g_first = p.cl[clu * 3], count = p.cl[clu * 3 + 1], blk_first = p.cl[clu * 3 + 2];
    const int nblk = (int)((count + NSB - 1) / NSB);
    int8_t *YS = p.YS + (int64_t)clu * p.nrb * 4 * HALF;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 2); }
        mbar_init(tfull, 1);
        mbar_init(tempty, 4);
        mbar_init(xbar, 1);
        mbar_init(yready, 2);
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

    if (warp == 4) {
        // ------------------------------------------------------------ producer: my operand, to both CTAs
        if (lane == 0) {
            uint32_t q = 0, yw = 0;
            bool lockstep = p.lag > 0;              // a performance hint only: given up if it ever stalls
            for (int b = 0; b < nblk; ++b) {
                for (int rb = 1; rb < p.nrb; ++rb) {
                    const int nch = 4 * rb;
                    const int8_t *Arow = p.LA + 2ll * rb * (rb + 1) * HALF;
                    const int64_t t = (int64_t)b * (p.nrb - 1) + rb - 1;
                    if (crank == 0 && lockstep && t >= p.lag) {
                        // wait (bounded: ~0.5 s, e.g. clusters not co-resident under MPS) until every
                        // cluster with step t - lag has issued it
                        const int64_t tw = t - p.lag;
                        const int need = p.need[tw / (p.nrb - 1)];
                        int v;
                        for (int spin = 0;; ++spin) {
                            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p.step_done + tw) : "memory");
                            if (v >= need) break;
                            if (spin > (1 << 21)) { lockstep = false; break; }
                            __nanosleep(200);
                        }
                    }
                    for (int c = 0; c < nch; ++c, ++q) {
                        if (crank == 1 && c == 4 * (rb - 1)) { mbar_wait_cluster(yready, yw & 1); ++yw; }
                        const int st = q % STAGES;
                        mbar_wait(&empty[st], ((q / STAGES) & 1) ^ 1);
                        uint8_t *dst = ring + st * STAGE;
                        mbar_arrive_expect_tx(&full[st], STAGE);
                        const int8_t *src = crank == 0 ? Arow + (int64_t)c * HALF : YS + (int64_t)c * HALF;
                        uint8_t *d = crank == 0 ? dst + HALF : dst;     // B (L) after A (Y)
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                                     " [%0], [%1], %2, [%3], %4;\n"
                                     ::"r"(smem_u32(d)), "l"(src), "r"(HALF), "r"(smem_u32(&full[st])), "h"((uint16_t)3) : "memory");
                    }
                    if (crank == 0 && p.lag > 0) atomicAdd(p.step_done + t, 1);   // also after giving up: others may wait
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer (18 products per chunk)
        uint32_t q = 0, fl = 0;
        constexpr uint32_t idesc = i8_idesc(RB);
        for (int b = 0; b < nblk; ++b) {
            for (int rb = 1; rb < p.nrb; ++rb) {
                const int nch = 4 * rb;
                for (int c = 0; c < nch; ++c, ++q) {
                    const bool fresh = (c % FLUSH) == 0;
                    const bool last = (c + 1) % FLUSH == 0 || c + 1 == nch;
                    if (fresh) {
                        mbar_wait(tempty, (fl & 1) ^ 1);      // the previous flush drained by warps 0-3
                        asm volatile("tcgen05.fence::after_thread_sync;\n");
                    }
                    const int st = q % STAGES;
                    mbar_wait(&full[st], (q / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(ring + st * STAGE), b0 = a0 + HALF;
#pragma unroll
                        for (int l = 0; l < 4; ++l) {
                            const int d = soz_level(crank, l);
                            for (int pp = 0; pp <= d; ++pp) {                // L slice pp, Y slice d - pp
                                const uint64_t da = oz_desc(a0 + (d - pp) * SLICE), db = oz_desc(b0 + pp * SLICE);
                                const uint32_t acc = (fresh && pp == 0) ? 0u : 1u;
                                asm volatile("{\n .reg .pred pp;\n setp.ne.u32 pp, %4, 0;\n"
                                             " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, pp;\n}\n"
                                             ::"r"(tmem + (uint32_t)(l * RB)), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                            }
                        }
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
                                     " [%0], %1;\n" ::"r"(smem_u32(&empty[st])), "h"((uint16_t)3) : "memory");
                        if (last)
                            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                                         ::"r"(smem_u32(tfull)) : "memory");
                    }
                    __syncwarp();
                    if (last) ++fl;
                }
            }
        }
    } else if ((warp >> 1) != crank) {
        // ------------------------------------------------------------ exchange: the peer's samples
        const int jj = (warp & 1) * 32 + lane;                 // the peer's local sample index
        const uint32_t peer_xbar = mapa_peer(smem_u32(xbar), (uint32_t)(crank ^ 1));
        uint32_t fl = 0;
        for (int b = 0; b < nblk; ++b) {
            for (int rb = 1; rb < p.nrb; ++rb) {
                double *X = p.xch + (((int64_t)clu * 2 + (crank ^ 1)) * 2 + (rb & 1)) * RB * CS;
                const int nf = (4 * rb + FLUSH - 1) / FLUSH;
                for (int f = 0; f < nf; ++f, ++fl) {
                    mbar_wait(tfull, fl & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n");
                    soz_drain(tmem, warp, crank, X, jj, f == 0);
                    asm volatile("tcgen05.fence::before_thread_sync;\n");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty);
                }
                __threadfence();
                named_sync(BAR_EX, 64);
                if (tid == ((crank ^ 1) * 64))                 // first exchange thread
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(peer_xbar) : "memory");
            }
        }
    } else {
        // ------------------------------------------------------------ chain: my 64 samples
        const int jj = (warp & 1) * 32 + lane;                 // local sample index
        const int m = crank * CS + jj;                         // sample within the block (TMEM lane)
        const int tid_ch = jj;
        const uint32_t yready1 = mapa_peer(smem_u32(yready), 1u);
        uint32_t fl = 0, xp = 0;
        for (int b = 0; b < nblk; ++b) {
            const int64_t off = (int64_t)b * NSB + m;
            const bool valid = off < count;
            const uint64_t g = (uint64_t)(g_first + (valid ? off : (int64_t)b * NSB));
            const uint64_t r = g / (uint64_t)p.N;
            const uint64_t jl = g - r * (uint64_t)p.N + 1ull;
            const int64_t blk = (blk_first + b) * 2 + crank;
            double ell = 0.0;
            for (int rb = 0; rb < p.nrb; ++rb) {
                const int64_t row0 = (int64_t)rb * RB;
#pragma unroll
                for (int h = 0; h < 2; ++h) {                   // a, G, 1 / L_kk, scale of the row block
                    const int t = jj + h * 64;
                    const int64_t k = row0 + t;
                    const bool in = k < p.n;
                    a_s[t] = in ? p.a[k] : 0.0;
                    G_s[t] = in ? p.G[k] : 0ull;
                    dinv[t] = in ? 1.0 / p.L[tile_offset(rb, rb) + (int64_t)t * kTile + t] : 1.0;
                    scl[t] = in ? p.rowscale[k] * 128.0 : 0.0;
                }
                if (rb == 0) {
                    for (int li = 0; li < RB; ++li) Ssm[li * CS + jj] = 0.0;
                } else {
                    const int nf = (4 * rb + FLUSH - 1) / FLUSH;
                    for (int f = 0; f < nf; ++f, ++fl) {
                        mbar_wait(tfull, fl & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;\n");
                        soz_drain(tmem, warp, crank, Ssm, jj, f == 0);
                        asm volatile("tcgen05.fence::before_thread_sync;\n");
                        __syncwarp();
                        if (lane == 0) mbar_arrive(tempty);
                    }
                    mbar_wait_cluster(xbar, xp & 1);            // the peer's levels for my samples
                    ++xp;
                    const double *X = p.xch + (((int64_t)clu * 2 + crank) * 2 + (rb & 1)) * RB * CS;
                    named_sync(BAR_CH, 64);                      // scl complete
                    for (int l0 = 0; l0 < RB; l0 += 16) {          // 16 loads in flight, then use
                        double xv[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) xv[i] = __ldcg(X + (l0 + i) * CS + jj);
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            Ssm[(l0 + i) * CS + jj] = (Ssm[(l0 + i) * CS + jj] + xv[i]) * scl[l0 + i];
                    }
                }
                named_sync(BAR_CH, 64);
                soz_chain_rowblock(p, smo, rb, jj, m, valid, r, jl, ell, YS, tid_ch);
                if (rb + 1 < p.nrb) {
                    asm volatile("fence.proxy.async.global;\n" ::: "memory");   // Y digits -> the TMA reads
                    __threadfence();
                    named_sync(BAR_CH, 64);
                    if (jj == 0)
                        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(yready1) : "memory");
                } else {
                    named_sync(BAR_CH, 64);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {                   // per-row (max, sum) of my 64 samples
                    const int t = jj + h * 64;
                    const int64_t k = row0 + t;
                    if (k < p.n) {
                        const double m0 = ps[(t * 2) * 2], s0 = ps[(t * 2) * 2 + 1];
                        const double m1 = ps[(t * 2 + 1) * 2], s1 = ps[(t * 2 + 1) * 2 + 1];
                        const double mm = fmax(m0, m1);
                        double ss = 0.0;
                        if (mm != -CUDART_INF) {
                            if (m0 != -CUDART_INF) ss += s0 * exp(m0 - mm);
                            if (m1 != -CUDART_INF) ss += s1 * exp(m1 - mm);
                        }
                        *reinterpret_cast<double2 *>(p.part + (blk * p.n_pad + k) * 2) = make_double2(mm, ss);
                    }
                }
                named_sync(BAR_CH, 64);                          // ps / a_s free for the next row block
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    cluster_sync_all();                                          // no CTA leaves while its peer may write into it
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
}

cudaError_t sov_oz_init() {
    return cudaFuncSetAttribute(k_sov_oz, cudaFuncAttributeMaxDynamicSharedMemorySize, soz::SMEM);
}

// Co-resident clusters of k_sov_oz (a cluster's two CTAs sit in one GPC; ~1 CTA per SM).
int sov_oz_max_clusters(int nsm) {
    static int cached = 0;
    if (!cached) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(soz::NT);
        cfg.dynamicSmemBytes = soz::SMEM;
        int v = 0;
        if (cudaOccupancyMaxActiveClusters(&v, k_sov_oz, &cfg) != cudaSuccess || v < 1) {
            cudaGetLastError();
            v = nsm / 2;
        }
        cached = std::min(v, nsm / 2);
    }
    return cached;
}

int64_t sov_oz_ys_bytes(int64_t n, int clusters) { return (int64_t)clusters * ((n + 127) / 128) * 4 * soz::HALF; }
int64_t sov_oz_xch_bytes(int clusters) { return (int64_t)clusters * 4 * soz::RB * soz::CS * 8; }

// Balanced partition of [g_begin, g_end) over clusters (blocks of 128 samples each).
int64_t sov_oz_partition(int64_t g_begin, int64_t g_end, int clusters, int64_t *cl) {
    const int64_t ns = g_end - g_begin, base = ns / clusters, rem = ns % clusters;
    int64_t blk = 0, g = g_begin;
    for (int c = 0; c < clusters; ++c) {
        const int64_t cnt = base + (c < rem ? 1 : 0);
        cl[3 * c] = g;
        cl[3 * c + 1] = cnt;
        cl[3 * c + 2] = blk;
        g += cnt;
        blk += (cnt + soz::NSB - 1) / soz::NSB;
    }
    return blk;
}

cudaError_t launch_sov_oz(const SovOzLaunch &L, cudaStream_t st) {
    SovOzArgs a;
    a.LA = L.LA; a.rowscale = L.rowscale; a.L = L.L; a.n = L.n; a.nrb = (int)((L.n + 127) / 128);
    a.n_pad = (int64_t)a.nrb * 128; a.a = L.a; a.G = L.G; a.N = L.N; a.seed = L.seed; a.cl = L.cl; a.YS = L.YS;
    a.xch = L.xch; a.part = L.part; a.flag = L.flag;
    a.lag = L.lag; a.step_done = L.step_done; a.need = L.need;
    cudaError_t e = cudaMemsetAsync(L.flag, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    if (a.lag > 0 && a.nrb > 1 &&
        (e = cudaMemsetAsync(L.step_done, 0, sizeof(int) * (size_t)L.max_blocks * (a.nrb - 1), st)) != cudaSuccess)
        return e;
    k_sov_oz<<<2 * L.clusters, soz::NT, soz::SMEM, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return launch_reduce_blocks(L.part, 2 * L.nblk, L.n, a.n_pad, L.Mout, L.Sout, st);
}

}  // namespace mvn
