// K5/K6 — the SOV sweep with Richtmyer-lattice QMC (Alg. 2 PMVN; Alg. 3 QMC tile
// kernel; Eq. 2-3), all prefixes in one sweep (reading R1).
//
// Work decomposition (B200-first, not the paper's tile-task DAG):
//   * The parallel axis is the sample ("MC chain"). A CTA owns a block of NB consecutive
//     global samples and sweeps all n rows in row blocks of 64; CTAs are persistent (one per SM).
//   * Row block r (rows [64r, 64r+64)):
//       (a6) S = L[rows, 0:64r] * Y[0:64r, block]  — left-looking fp64 DMMA GEMM (box (c), one
//            product serves a' and b', reading R7), operands streamed by a 3-stage cp.async
//            pipeline: L panel from L2 (all CTAs sweep the same rows), Y history from this CTA's
//            HBM scratch.
//       (a7) the in-block recursion of Alg. 3 per sample (thread j = sample j): in sub-blocks of
//            8 rows, s += in-block dot, Phi/Phi^{-1} step (normal.cuh), log-weight ell += log q,
//            y written to the Y history (coalesced) and folded into the remaining rows of S.
//       (a8) per-row log-sum-exp over the block's samples (warp shuffles) -> (M, S) partial per
//            (sample block, row).
//   * k_reduce_blocks combines the block partials of every prefix in fixed order (deterministic).
// The lattice point w (reading R8) is generated in registers from 64-bit integers; the n x NR
// matrices R, A, B of Alg. 2 are never materialised.
#include "common.cuh"
#include "gemm_dmma.cuh"
#include "mvn_internal.h"
#include "normal.cuh"

namespace mvn {
namespace sovk {
constexpr int M = 64;              // SOV row block
constexpr int BK = 16, STAGES = 3;
constexpr int SA = M + 4;          // 68 == 4 (mod 16)
constexpr int NT = 256;            // threads per CTA
template <int NB> struct Cfg {
    static constexpr int SB = NB + 4;      // pipeline B stride, == 4 (mod 16) for NB % 16 == 0
    static constexpr int SS = NB + 8;      // S / ell tile stride (16-byte stores conflict-free)
    static constexpr int WN = NB / 32;     // 8-column DMMA blocks per warp (warp tile 32 x NB/4)
    static constexpr int PIPE = STAGES * BK * (SA + SB);
    static constexpr int UNION = (PIPE > M * SS) ? PIPE : M * SS;
    static constexpr int SMEM = (UNION + M * M + 3 * M) * 8;
};
}  // namespace sovk

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
    int nrb;                 // row blocks of 64 (ceil(n/64))
    const double *a, *b;     // b may be null (+inf)
    const uint64_t *G;
    int64_t N;
    uint64_t seed;
    int64_t g_begin, g_end;  // global sample range
    int64_t nblk;            // sample blocks
    int64_t n_pad;           // Y-history rows per slot (nrb*64)
    double *Y;               // [gridDim][n_pad][NB]
    double *part;            // [nblk][n_pad][2]
};

template <int NB, bool HAS_B>
__global__ void __launch_bounds__(sovk::NT, 1) k_sov(SovArgs p) {
    using namespace sovk;
    using C = Cfg<NB>;
    extern __shared__ double sm[];
    double *As = sm;                                    // pipeline (union with S)
    double *Bs = sm + STAGES * BK * SA;
    double *S = sm;                                     // M x SS: s, then ell
    double *Ld = sm + C::UNION;                         // 64 x 64 diagonal block of L, row-major
    double *a_s = Ld + M * M;
    double *b_s = a_s + M;
    uint64_t *G_s = reinterpret_cast<uint64_t *>(b_s + M);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp & 1) * 32, wn0 = (warp >> 1) * (NB / 4);
    double *Yslot = p.Y + (int64_t)blockIdx.x * p.n_pad * NB;

    for (int64_t blk = blockIdx.x; blk < p.nblk; blk += gridDim.x) {
        const int64_t g0 = p.g_begin + blk * NB;
        const int64_t rem = p.g_end - g0;
        const int cnt = rem < NB ? (int)rem : NB;
        const int j = tid;                               // sample within block (tid < NB)
        const uint64_t g = (uint64_t)(g0 + (j < NB ? j : 0));
        const uint64_t r = g / (uint64_t)p.N;
        const uint64_t jl = g - r * (uint64_t)p.N + 1ull;   // 1-based lattice index
        double ell = 0.0;

        for (int rb = 0; rb < p.nrb; ++rb) {
            const int64_t row0 = (int64_t)rb * M;
            const int R = (int)(row0 / kTile), hh = (int)(row0 % kTile);
            // ---------------------------------------------------------------- (a6) GEMM
            if (rb > 0) {
                double acc[4][C::WN][2];
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < C::WN; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
                auto load = [&](int ch, int st) {
                    const int64_t kc = (int64_t)ch * BK;              // first column of the chunk
                    const int T = (int)(kc / kTile), cc = (int)(kc % kTile);
                    const double *Lsrc = p.L + tile_offset(R, T) + (int64_t)cc * kTile + hh;
                    double *as = As + st * BK * SA;
                    double *bs = Bs + st * BK * C::SB;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {                     // 16 cols x 64 rows
                        const int e = q * NT + tid;
                        const int col = e >> 5, seg = e & 31;
                        cp_async16(as + col * SA + seg * 2, Lsrc + (int64_t)col * kTile + seg * 2);
                    }
                    const double *Ysrc = Yslot + kc * NB;               // 16 rows x NB, contiguous
#pragma unroll
                    for (int q = 0; q < NB / 32; ++q) {
                        const int e = q * NT + tid;
                        const int row = e / (NB / 2), seg = e % (NB / 2);
                        cp_async16(bs + row * C::SB + seg * 2, Ysrc + (int64_t)row * NB + seg * 2);
                    }
                };
                gemm_mainloop<BK, STAGES, SA, C::SB, 4, C::WN>((int)(row0 / BK), As, Bs, wm0, wn0, lane, acc, load);
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    const int row = wm0 + x * 8 + (lane >> 2);
#pragma unroll
                    for (int y = 0; y < C::WN; ++y) {
                        const int col = wn0 + y * 8 + 2 * (lane & 3);
                        *reinterpret_cast<double2 *>(S + row * C::SS + col) = make_double2(acc[x][y][0], acc[x][y][1]);
                    }
                }
            } else {
                for (int e = tid; e < M * C::SS; e += NT) S[e] = 0.0;
            }
            // diagonal block L[row0:+64, row0:+64] (row-major in smem), limits, generators
            {
                const double *Dsrc = p.L + tile_offset(R, R) + (int64_t)hh * kTile + hh;
                for (int e = tid; e < M * M; e += NT) {
                    const int col = e >> 6, row = e & 63;            // coalesced along rows
                    Ld[row * M + col] = Dsrc[(int64_t)col * kTile + row];
                }
                if (tid < M) {
                    const int64_t k = row0 + tid;
                    a_s[tid] = k < p.n ? p.a[k] : 0.0;
                    b_s[tid] = (HAS_B && k < p.n) ? p.b[k] : CUDART_INF;
                    G_s[tid] = k < p.n ? p.G[k] : 0ull;
                }
            }
            __syncthreads();
            // ---------------------------------------------------------------- (a7) chain
            if (j < NB) {
#pragma unroll 1
                for (int sb = 0; sb < M / 8; ++sb) {
                    const int rb0 = sb * 8;
                    double s[8], yv[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) s[i] = S[(rb0 + i) * C::SS + j];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int li = rb0 + i;
                        const int64_t k = row0 + li;
                        double y = 0.0;
                        if (k < p.n) {
                            const double lkk = Ld[li * M + li];
                            const double ap = (a_s[li] - s[i]) / lkk;
                            const double w = lattice_w(jl, G_s[li], lattice_shift(p.seed, r, (uint64_t)k));
                            double lq;
                            if (HAS_B) sov_step(ap, (b_s[li] - s[i]) / lkk, w, lq, y);
                            else sov_step_upper(ap, w, lq, y);
                            ell += lq;
                        }
                        yv[i] = y;
                        S[li * C::SS + j] = ell;
                        Yslot[k * NB + j] = y;
#pragma unroll
                        for (int i2 = i + 1; i2 < 8; ++i2) s[i2] += Ld[(rb0 + i2) * M + li] * y;
                    }
                    for (int li = rb0 + 8; li < M; ++li) {
                        double t = S[li * C::SS + j];
#pragma unroll
                        for (int i = 0; i < 8; ++i) t += Ld[li * M + rb0 + i] * yv[i];
                        S[li * C::SS + j] = t;
                    }
                }
            }
            __threadfence_block();
            __syncthreads();
            // ---------------------------------------------------------------- (a8) per-row lse
            for (int li = warp; li < M; li += NT / 32) {
                const int64_t k = row0 + li;
                if (k >= p.n) break;
                double m = -CUDART_INF;
                for (int jj = lane; jj < cnt; jj += 32) m = fmax(m, S[li * C::SS + jj]);
#pragma unroll
                for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
                double sum = 0.0;
                if (m != -CUDART_INF)
                    for (int jj = lane; jj < cnt; jj += 32) sum += exp(S[li * C::SS + jj] - m);
#pragma unroll
                for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                if (lane == 0)
                    *reinterpret_cast<double2 *>(p.part + (blk * p.n_pad + k) * 2) = make_double2(m, sum);
            }
            __syncthreads();
        }
    }
}

// K6: combine block partials per prefix in ascending block order.
__global__ void k_reduce_blocks(const double *__restrict__ part, int64_t nblk, int64_t n, int64_t n_pad,
                                double *__restrict__ Mo, double *__restrict__ So) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    double m = -CUDART_INF;
    for (int64_t b = 0; b < nblk; ++b) m = fmax(m, part[(b * n_pad + k) * 2]);
    double s = 0.0;
    if (m != -CUDART_INF)
        for (int64_t b = 0; b < nblk; ++b) {
            const double mb = part[(b * n_pad + k) * 2], sb = part[(b * n_pad + k) * 2 + 1];
            if (mb != -CUDART_INF) s += sb * exp(mb - m);
        }
    Mo[k] = m;
    So[k] = s;
}

template <int NB, bool HB>
static cudaError_t set_attr() {
    return cudaFuncSetAttribute(k_sov<NB, HB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sovk::Cfg<NB>::SMEM);
}

cudaError_t sov_init() {
    cudaError_t e = cudaSuccess;
#define MVN_SOV_ATTR(NB)                               \
    if ((e = set_attr<NB, false>()) != cudaSuccess) return e; \
    if ((e = set_attr<NB, true>()) != cudaSuccess) return e;
    MVN_SOV_ATTR(128) MVN_SOV_ATTR(160) MVN_SOV_ATTR(192) MVN_SOV_ATTR(224) MVN_SOV_ATTR(256)
#undef MVN_SOV_ATTR
    return e;
}

int sov_pick_nb(int64_t nsamp, int64_t n, int nsm) {
    static const int cand[5] = {256, 224, 192, 160, 128};
    int best = 256;
    double bestc = 1e300;
    const double chain = (double)((n + 63) / 64) * 64.0 * 1500.0;   // latency-bound chain clk per block
    for (int c : cand) {
        const int64_t nblk = (nsamp + c - 1) / c;
        const int64_t waves = (nblk + nsm - 1) / nsm;
        const double gemm = (double)c * (double)n * (double)n / 128.0;  // DMMA clk per block at full rate
        const double cost = (double)waves * (gemm + chain);
        if (cost < bestc * (1 - 1e-9)) { bestc = cost; best = c; }
    }
    return best;
}

size_t sov_smem_bytes(int nb) {
    switch (nb) {
        case 128: return sovk::Cfg<128>::SMEM;
        case 160: return sovk::Cfg<160>::SMEM;
        case 192: return sovk::Cfg<192>::SMEM;
        case 224: return sovk::Cfg<224>::SMEM;
        default: return sovk::Cfg<256>::SMEM;
    }
}

cudaError_t launch_sov(const SovLaunch &L, cudaStream_t st) {
    SovArgs a;
    a.L = L.L; a.n = L.n; a.nrb = (int)((L.n + 63) / 64); a.a = L.a; a.b = L.b; a.G = L.G; a.N = L.N;
    a.seed = L.seed; a.g_begin = L.g_begin; a.g_end = L.g_end; a.nblk = L.nblk; a.n_pad = (int64_t)a.nrb * 64;
    a.Y = L.Y; a.part = L.part;
    const dim3 grid(L.grid), block(sovk::NT);
    const size_t sm = sov_smem_bytes(L.nb);
#define MVN_SOV_LAUNCH(NB)                                                               \
    case NB:                                                                             \
        if (L.b) k_sov<NB, true><<<grid, block, sm, st>>>(a);                            \
        else k_sov<NB, false><<<grid, block, sm, st>>>(a);                               \
        break;
    switch (L.nb) {
        MVN_SOV_LAUNCH(128) MVN_SOV_LAUNCH(160) MVN_SOV_LAUNCH(192) MVN_SOV_LAUNCH(224) MVN_SOV_LAUNCH(256)
        default: return cudaErrorInvalidValue;
    }
#undef MVN_SOV_LAUNCH
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_reduce_blocks<<<(unsigned)((L.n + 255) / 256), 256, 0, st>>>(L.part, L.nblk, L.n, a.n_pad, L.Mout, L.Sout);
    return cudaGetLastError();
}

}  // namespace mvn
