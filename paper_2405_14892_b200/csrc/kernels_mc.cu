// NEXT-2 — Monte-Carlo validation of the confidence regions (§V-C1 blue text, P:595:
// "draws N samples from the fitted distribution, where N_s represents the number of samples
// exceeding a given threshold ... p_hat(alpha) = N_s/N"; supplement P:20-23).
//
// In the sorted order of the sweep, a field draw is X = mu + L z, so X_{o(k)} > u  <=>  (L z)_k > a_k
// with a_k = u - mu_{o(k)} (reading R2). A region for level 1-alpha is a prefix o(1..k*), so one
// draw counts for EVERY level at once through its first failing row f = min{k : (L z)_k <= a_k}
// (n if none): the sample exceeds on region k* iff f >= k*. Hence
//   K7 k_mc_gen  : z_{k,s} = Phi^{-1}(w), w from a counter hash of (seed, s, k) (reading R20), into a
//                  padded [sample block][n_pad][SZ] buffer;
//   K8 k_mc_trmm : X = L Z on fp64 DMMA (L lower tile-packed; the row tile i needs tiles 0..i),
//                  persistent, producer warp + 8 DMMA warps as in the Cholesky update kernel; the
//                  epilogue never stores X — it reduces each sample column of the 128 x 128 tile to
//                  its first failing row and atomicMin's it into first[s];
//   K9 k_mc_count: count[first[s]] += 1 (histogram over 0..n).
// Algorithmic work: n(n+1) flops per sample for L z (one FMA per (k, t <= k)).
#include <algorithm>
#include <climits>

#include "common.cuh"
#include "mvn_internal.h"
#include "normal.cuh"

namespace mvn {
namespace mck {
constexpr int BK = 8, STAGES = 4;
constexpr int SP = kTile + 4;                 // 132: padded smem row (conflict-free fragments)
constexpr int SZ = kTile + 4;                 // Z row stride in HBM (one bulk copy per chunk)
constexpr int STAGE = 2 * BK * SP;
constexpr int NCONS = 256, NT = NCONS + 32;
constexpr int OFF_BAR = STAGES * STAGE;
constexpr int SMEM = (OFF_BAR + 2 * STAGES) * 8;
constexpr int CPT = kTile / BK;               // K-chunks per tile
}  // namespace mck

__device__ __forceinline__ uint64_t mc_mix(uint64_t seed, uint64_t s, uint64_t k) {
    // SplitMix64 output function of the counter seed + GAMMA * (s * 2^32 + k + 1) (reading R20,
    // the same construction as the lattice shifts of R8 with the sample index in place of r)
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * ((s << 32) + k + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// K7: Z[sb][k][j] = Phi^{-1}(w(seed, s0 + sb*128 + j, k)); rows >= n and samples >= ns are zero.
__global__ void __launch_bounds__(256) k_mc_gen(double *__restrict__ Z, int64_t n, int64_t n_pad, int64_t s0, int64_t ns,
                                                uint64_t seed, int64_t ez) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // over [sb][n_pad][128]
    if (e >= ez) return;
    const int j = (int)(e & (kTile - 1));
    const int64_t rk = e >> 7;
    const int64_t k = rk % n_pad, sb = rk / n_pad;
    const int64_t s = sb * kTile + j;
    double z = 0.0;
    if (k < n && s < ns) {
        const uint64_t X = mc_mix(seed, (uint64_t)(s0 + s), (uint64_t)k);
        const double w = ((double)(X >> 12) + 0.5) * 0x1p-52;
        z = (w <= 0.5) ? Phi_inv_lower(w) : -Phi_inv_lower(1.0 - w);   // 1 - w exact (R8)
    }
    Z[(sb * n_pad + k) * mck::SZ + j] = z;
}

__device__ __forceinline__ void cp_async16_mc(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}

// K8. Items (row tile i, sample block sb), heaviest rows first: item -> i = nt-1 - item / nsb.
__global__ void __launch_bounds__(mck::NT, 1) k_mc_trmm(const double *__restrict__ tiles, int64_t n, int nt,
                                                         const double *__restrict__ Z, int64_t n_pad, int nsb, int64_t ns,
                                                         const double *__restrict__ a, int *__restrict__ first) {
    using namespace mck;
    extern __shared__ double sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + OFF_BAR);
    uint64_t *empty = full + STAGES;
    const int tid = threadIdx.x;
    const int64_t nitems = (int64_t)nt * nsb;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCONS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    uint32_t q = 0;
    if (tid >= NCONS) {
        // ------------------------------------------------------------ producer warp
        const int lane = tid & 31;
        for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
            const int i = nt - 1 - (int)(item / nsb), sb = (int)(item % nsb);
            const double *Lrow = tiles + tile_offset(i, 0);          // row panel i: tiles (i, 0..i) contiguous
            const double *Zb = Z + (int64_t)sb * n_pad * SZ;
            const int nch = (i + 1) * CPT;
            for (int c = 0; c < nch; ++c, ++q) {
                const int st = q % STAGES;
                mbar_wait(&empty[st], ((q / STAGES) & 1) ^ 1);
                double *as = sm + st * STAGE;
                double *bs = as + BK * SP;
                const double *a0 = Lrow + (int64_t)c * BK * kTile + lane * 2;   // 8 columns (1 KB each)
#pragma unroll
                for (int t = 0; t < BK; ++t)
#pragma unroll
                    for (int h = 0; h < 2; ++h) cp_async16_mc(as + t * SP + h * 64 + lane * 2, a0 + (int64_t)t * kTile + h * 64);
                cp_async_mbar_arrive(&full[st]);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[st], BK * SZ * 8);
                    bulk_g2s(bs, Zb + (int64_t)c * BK * SZ, BK * SZ * 8, &full[st]);
                }
            }
        }
        return;
    }
    // ---------------------------------------------------------------- DMMA warps
    const int lane = tid & 31, warp = tid >> 5;
    const int wn0 = warp * 16;                       // 16 sample columns per warp, all 128 rows
    for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
        const int i = nt - 1 - (int)(item / nsb), sb = (int)(item % nsb);
        const int nch = (i + 1) * CPT;
        double acc[16][2][2];
#pragma unroll
        for (int x = 0; x < 16; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
        for (int c = 0; c < nch; ++c, ++q) {
            const int st = q % STAGES;
            mbar_wait(&full[st], (q / STAGES) & 1);
            const double *as = sm + st * STAGE;
            const double *bs = as + BK * SP;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double fa[16], fb[2];
                const int kr = kk + (lane & 3);
#pragma unroll
                for (int y = 0; y < 2; ++y) fb[y] = bs[kr * SP + wn0 + y * 8 + (lane >> 2)];
#pragma unroll
                for (int x = 0; x < 16; ++x) fa[x] = as[kr * SP + x * 8 + (lane >> 2)];
#pragma unroll
                for (int x = 0; x < 16; ++x)
#pragma unroll
                    for (int y = 0; y < 2; ++y) dmma(acc[x][y][0], acc[x][y][1], fa[x], fb[y]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        // epilogue: thread holds rows x*8 + lane/4 (x < 16) of columns wn0 + y*8 + 2(lane%4) + e
        int fmin[2][2] = {{INT_MAX, INT_MAX}, {INT_MAX, INT_MAX}};
#pragma unroll
        for (int x = 15; x >= 0; --x) {
            const int64_t row = (int64_t)i * kTile + x * 8 + (lane >> 2);
            if (row < n) {
                const double ar = __ldg(a + row);
#pragma unroll
                for (int y = 0; y < 2; ++y)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (!(acc[x][y][e] > ar)) fmin[y][e] = (int)row;
            }
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1)
#pragma unroll
            for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int e = 0; e < 2; ++e) fmin[y][e] = min(fmin[y][e], __shfl_xor_sync(0xffffffffu, fmin[y][e], o));
        if (lane < 4) {
#pragma unroll
            for (int y = 0; y < 2; ++y)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int64_t s = (int64_t)sb * kTile + wn0 + y * 8 + 2 * lane + e;
                    if (s < ns && fmin[y][e] != INT_MAX) atomicMin(first + s, fmin[y][e]);
                }
        }
    }
}

__global__ void k_mc_init(int *__restrict__ first, int64_t ns, int n) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s < ns) first[s] = n;
}

// K9: count[f] += 1 for every sample (f in 0..n).
__global__ void k_mc_count(const int *__restrict__ first, int64_t ns, unsigned long long *__restrict__ count) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s < ns) atomicAdd(count + first[s], 1ull);
}

cudaError_t launch_mc_first_init(int *first, int64_t ns, int n, cudaStream_t st) {
    k_mc_init<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(first, ns, n);
    return cudaGetLastError();
}

cudaError_t launch_mc_count(const int *first, int64_t ns, unsigned long long *count, cudaStream_t st) {
    k_mc_count<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(first, ns, count);
    return cudaGetLastError();
}

cudaError_t mc_init() {
    return cudaFuncSetAttribute(k_mc_trmm, cudaFuncAttributeMaxDynamicSharedMemorySize, mck::SMEM);
}

int64_t mc_z_doubles(int64_t n, int64_t ns) {
    const int64_t n_pad = (n + kTile - 1) / kTile * kTile;
    return (ns + kTile - 1) / kTile * n_pad * mck::SZ;
}

// One chunk of ns samples starting at global sample s0: Z generation, TRMM + first failure,
// histogram into count (accumulated).
cudaError_t launch_mc_chunk(int64_t n, const double *tiles, const double *a, uint64_t seed, int64_t s0, int64_t ns,
                            double *Z, int *first, unsigned long long *count, int nsm, cudaStream_t st) {
    const int nt = (int)((n + kTile - 1) / kTile);
    const int64_t n_pad = (int64_t)nt * kTile;
    const int nsb = (int)((ns + kTile - 1) / kTile);
    const int64_t ez = (int64_t)nsb * n_pad * kTile;
    k_mc_gen<<<(unsigned)((ez + 255) / 256), 256, 0, st>>>(Z, n, n_pad, s0, ns, seed, ez);
    k_mc_init<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(first, ns, (int)n);
    const int64_t items = (int64_t)nt * nsb;
    const int grid = (int)std::min<int64_t>(items, nsm);
    k_mc_trmm<<<grid, mck::NT, mck::SMEM, st>>>(tiles, n, nt, Z, n_pad, nsb, ns, a, first);
    k_mc_count<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(first, ns, count);
    return cudaGetLastError();
}

}  // namespace mvn
