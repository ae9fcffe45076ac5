// Feasibility probe (tooling, not product) for the round-2 int8 SOV design: a
// 2-CTA cluster computes D[128 x N] = A[128 x K] * B[N x K]^T with ONE tcgen05.mma.cta_group::2
// .kind::i8 of M = 128 (each CTA holds 64 rows of A and N/2 rows of B in its shared memory, and 64
// rows of D in its TMEM). Questions: (1) which TMEM lanes hold a CTA's 64 rows (read all 128 lanes
// back and match them against the CPU product), (2) the int8 MAC rate per SM of this shape — the
// tcgen05 floor max(M,128) N / (256 cta_group) predicts the full M128 N128 cta_group::1 rate per SM
// with only 64 rows per CTA (cta_group::1 M64 runs at half rate, tools/umma_i8_m64.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_i8_2sm tools/umma_i8_2sm.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// kind::i8, D s32, A/B signed, K-major, N>>3 at [17,23), M>>4 at [24,29) (M = 128: the pair's rows)
__host__ __device__ constexpr uint32_t make_idesc(int n, int m) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ int core_off(int row, int k, int K) {
    return (((row >> 3) * (K >> 4) + (k >> 4)) << 7) + ((row & 7) << 4) + (k & 15);
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_umma_2sm(const int8_t *A, const int8_t *B, int K, int reps, int32_t *D, long long *cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    int8_t *As = reinterpret_cast<int8_t *>(sm);          // 64 rows x K
    int8_t *Bs = As + 64 * K;                              // N/2 rows x K
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    for (int e = tid; e < 64 * K; e += 128) As[core_off(e / K, e % K, K)] = A[(int64_t)(64 * rank + e / K) * K + e % K];
    for (int e = tid; e < (N / 2) * K; e += 128) Bs[core_off(e / K, e % K, K)] = B[(int64_t)((N / 2) * rank + e / K) * K + e % K];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(N < 32 ? 32 : N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    constexpr uint32_t idesc = make_idesc(N, 128);
    long long t0 = clock64();
    if (rank == 0 && tid == 0) {
        const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs);
        const uint32_t sbo = (K >> 4) << 7;
        for (int r = 0; r < reps; ++r)
            for (int k = 0; k < K; k += 32) {
                const uint64_t da = make_desc(a0 + (k >> 4) * 128, 128, sbo);
                const uint64_t db = make_desc(b0 + (k >> 4) * 128, 128, sbo);
                const uint32_t acc = (r > 0 || k > 0) ? 1u : 0u;
                asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n"
                             " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                     ::"r"(smem_u32(&mbar)), "h"((uint16_t)3) : "memory");
    }
    asm volatile("{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(smem_u32(&mbar)) : "memory");
    long long t1 = clock64();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    for (int c = 0; c < N; c += 8) {
        uint32_t v[8];
        const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        for (int j = 0; j < 8; ++j) D[((int64_t)rank * 128 + warp * 32 + lane) * N + c + j] = (int32_t)v[j];
    }
    if (rank == 0 && tid == 0) cycles[0] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(N < 32 ? 32 : N));
}

template <int N>
int run(int K, int reps) {
    std::vector<int8_t> A(128 * K), B(N * K);
    srand(11);
    for (auto &x : A) x = (int8_t)(rand() % 255 - 127);
    for (auto &x : B) x = (int8_t)(rand() % 255 - 127);
    int8_t *dA, *dB; int32_t *dD; long long *dc;
    cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, 2 * 128 * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 2 * 128 * N * 4);
    const int smem = (64 + N / 2) * K;
    cudaFuncSetAttribute(k_umma_2sm<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_umma_2sm<N><<<2, 128, smem>>>(dA, dB, K, reps, dD, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"N\":%d,\"err\":\"%s\"}\n", N, cudaGetErrorString(e)); return 1; }
    std::vector<int32_t> D(2 * 128 * N);
    long long cyc;
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    std::vector<int32_t> R(128 * N);
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
            long long s = 0;
            for (int k = 0; k < K; ++k) s += (long long)A[i * K + k] * B[j * K + k];
            R[i * N + j] = (int32_t)(s * reps);
        }
    // lane -> row map per CTA: the reference row whose N values equal the lane's
    int matched = 0;
    printf("{\"N\":%d,\"K\":%d,\"reps\":%d,\"cycles\":%lld,\"mac_per_clk_per_sm\":%.1f,\"lanes\":[", N, K, reps, cyc,
           128.0 * N * K * reps / (double)cyc / 2.0);
    for (int cta = 0; cta < 2; ++cta)
        for (int l = 0; l < 128; ++l) {
            int row = -1;
            for (int i = 0; i < 128 && row < 0; ++i) {
                bool eq = true;
                for (int j = 0; j < N && eq; ++j) eq = D[(cta * 128 + l) * N + j] == R[i * N + j];
                if (eq) row = i;
            }
            if (row >= 0) { ++matched; printf("%s[%d,%d,%d]", matched > 1 ? "," : "", cta, l, row); }
        }
    printf("],\"matched_lanes\":%d}\n", matched);
    if (matched == 0 && reps == 1) {            // diagnose: where do single values come from?
        const int probe[8] = {0, 1, 15, 16, 32, 63, 64, 127};
        for (int cta = 0; cta < 2; ++cta)
            for (int pi = 0; pi < 8; ++pi) {
                const int l = probe[pi];
                printf("  cta %d lane %3d:", cta, l);
                for (int j = 0; j < 4; ++j) {
                    const int32_t v = D[(cta * 128 + l) * N + j];
                    int fr = -1, fc = -1;
                    for (int i = 0; i < 128 && fr < 0; ++i)
                        for (int c = 0; c < N; ++c)
                            if (R[i * N + c] == v && v != 0) { fr = i; fc = c; break; }
                    printf(" %d(r%d,c%d)", v, fr, fc);
                }
                printf("\n");
            }
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
    return matched == 128 ? 0 : 1;
}

int main() {
    int fails = 0;
    fails += run<64>(64, 1);
    fails += run<128>(128, 1);
    fails += run<64>(512, 64);      // rate, operands resident in shared memory
    fails += run<128>(512, 64);
    fails += run<256>(256, 64);
    return fails;
}
