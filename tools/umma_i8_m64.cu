// Probe (tooling): tcgen05.mma.kind::i8 with M = 64, N = 128 — rate, and the TMEM placement of two
// M = 64 accumulators interleaved in the lane halves (second one at lane offset 16), as CUTLASS's
// tmem_frg "Interleaved" layout describes (row r of an M = 64 accumulator -> lane 32 (r / 16) + r % 16).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_i8_m64 tools/umma_i8_m64.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 64, N = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
           ((uint64_t)1 << 46);
}
constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
__device__ __forceinline__ int core_off(int row, int k, int K) { return (((row >> 3) * (K >> 4) + (k >> 4)) << 7) + ((row & 7) << 4) + (k & 15); }

// D0 = A0 B^T and D1 = A1 B^T (two accumulators, lane halves), reps times over K
__global__ void __launch_bounds__(128, 1) k_m64(const int8_t *A0, const int8_t *A1, const int8_t *B, int K, int reps, int32_t *D0,
                                                 int32_t *D1, long long *cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    int8_t *As0 = reinterpret_cast<int8_t *>(sm), *As1 = As0 + M * K, *Bs = As1 + M * K;
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < M * K; e += 128) { As0[core_off(e / K, e % K, K)] = A0[e]; As1[core_off(e / K, e % K, K)] = A1[e]; }
    for (int e = tid; e < N * K; e += 128) Bs[core_off(e / K, e % K, K)] = B[e];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    long long t0 = clock64();
    if (tid == 0) {
        const uint32_t a0 = smem_u32(As0), a1 = smem_u32(As1), b0 = smem_u32(Bs), sbo = (K >> 4) << 7;
        for (int r = 0; r < reps; ++r)
            for (int k = 0; k < K; k += 32) {
                const uint64_t db = make_desc(b0 + (k >> 4) * 128, 128, sbo);
                const uint32_t acc = (r > 0 || k > 0) ? 1u : 0u;
                asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tmem), "l"(make_desc(a0 + (k >> 4) * 128, 128, sbo)), "l"(db), "r"(idesc), "r"(acc));
                asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tmem + (16u << 16)), "l"(make_desc(a1 + (k >> 4) * 128, 128, sbo)), "l"(db), "r"(idesc), "r"(acc));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)) : "memory");
    }
    asm volatile("{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(smem_u32(&mbar)) : "memory");
    long long t1 = clock64();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // lane l of warp w: l < 16 -> D0 row 16 w + l; l >= 16 -> D1 row 16 w + l - 16
    for (int c = 0; c < N; c += 8) {
        uint32_t v[8];
        const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        int32_t *D = lane < 16 ? D0 : D1;
        const int row = warp * 16 + (lane & 15);
        for (int j = 0; j < 8; ++j) D[row * N + c + j] = (int32_t)v[j];
    }
    if (tid == 0) cycles[0] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(128));
}

int main() {
    const int K = 512, reps = 64;
    std::vector<int8_t> A0(M * K), A1(M * K), B(N * K);
    srand(11);
    for (auto &x : A0) x = (int8_t)(rand() % 255 - 127);
    for (auto &x : A1) x = (int8_t)(rand() % 255 - 127);
    for (auto &x : B) x = (int8_t)(rand() % 255 - 127);
    int8_t *dA0, *dA1, *dB; int32_t *dD0, *dD1; long long *dc;
    cudaMalloc(&dA0, A0.size()); cudaMalloc(&dA1, A1.size()); cudaMalloc(&dB, B.size());
    cudaMalloc(&dD0, M * N * 4); cudaMalloc(&dD1, M * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dA0, A0.data(), A0.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dA1, A1.data(), A1.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    const int smem = (2 * M + N) * K;
    cudaFuncSetAttribute(k_m64, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rr : {1, reps}) {
        k_m64<<<1, 128, smem>>>(dA0, dA1, dB, K, rr, dD0, dD1, dc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("{\"err\":\"%s\"}\n", cudaGetErrorString(e)); return 1; }
        std::vector<int32_t> D0(M * N), D1(M * N);
        long long cyc;
        cudaMemcpy(D0.data(), dD0, D0.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(D1.data(), dD1, D1.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
        long long bad0 = 0, bad1 = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                long long s0 = 0, s1 = 0;
                for (int k = 0; k < K; ++k) { s0 += (long long)A0[i * K + k] * B[j * K + k]; s1 += (long long)A1[i * K + k] * B[j * K + k]; }
                if ((int32_t)(s0 * rr) != D0[i * N + j]) ++bad0;
                if ((int32_t)(s1 * rr) != D1[i * N + j]) ++bad1;
            }
        printf("{\"M\":64,\"N\":128,\"K\":%d,\"reps\":%d,\"bad0\":%lld,\"bad1\":%lld,\"cycles\":%lld,\"mac_per_clk\":%.1f}\n", K, rr, bad0,
               bad1, cyc, 2.0 * M * N * K * rr / (double)cyc);
    }
    return 0;
}
