// Feasibility probe (tooling, not product): one CTA computes D[128 x N] = A[128 x K] * B[N x K]^T in
// int8 x int8 -> int32 with tcgen05.mma.kind::i8 (accumulator in TMEM, operands in shared memory,
// no-swizzle K-major canonical layout), reads D back with tcgen05.ld and compares with the CPU.
// Then times a long K loop (operands resident in smem) to get the per-SM int8 MMA rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/umma_i8_test tools/umma_i8_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Shared-memory matrix descriptor (sm_100 UMMA): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 [46,48), base offset 0, lbo mode 0, layout SWIZZLE_NONE (0) [61,64).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// Instruction descriptor, kind::i8: D s32 (c_format 2 at [4,6)), A/B signed (1 at [7,10), [10,13)),
// K-major A and B, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t make_idesc(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Canonical no-swizzle K-major layout: core matrix = 8 rows x 16 bytes (128 B contiguous, row r at
// 16 r). Core (g, kg) of a [rows][K] operand at ((g * (K/16)) + kg) * 128 bytes: LBO (next core in K)
// = 128 B, SBO (next 8-row group) = (K/16) * 128 B.
__device__ __forceinline__ int core_off(int row, int k, int K) {
    return (((row >> 3) * (K >> 4) + (k >> 4)) << 7) + ((row & 7) << 4) + (k & 15);
}

template <int N>
__global__ void __launch_bounds__(128, 1) k_umma_i8(const int8_t *A, const int8_t *B, int K, int reps, int32_t *D,
                                                     long long *cycles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    int8_t *As = reinterpret_cast<int8_t *>(sm);
    int8_t *Bs = As + M * K;
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < M * K; e += 128) As[core_off(e / K, e % K, K)] = A[e];
    for (int e = tid; e < N * K; e += 128) Bs[core_off(e / K, e % K, K)] = B[e];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)), "n"(N < 32 ? 32 : N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // operand stores -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    constexpr uint32_t idesc = make_idesc(N);
    long long t0 = clock64();
    if (tid == 0) {
        const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs);
        const uint32_t sboA = (K >> 4) << 7, sboB = (K >> 4) << 7;
        for (int r = 0; r < reps; ++r)
            for (int k = 0; k < K; k += 32) {
                const uint64_t da = make_desc(a0 + (k >> 4) * 128, 128, sboA);
                const uint64_t db = make_desc(b0 + (k >> 4) * 128, 128, sboB);
                const uint32_t acc = (r > 0 || k > 0) ? 1u : 0u;
                asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %4, 0;\n"
                             " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)) : "memory");
    }
    // wait for the MMAs
    asm volatile("{\n .reg .pred p;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(smem_u32(&mbar)) : "memory");
    long long t1 = clock64();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // TMEM -> registers: warp w owns lanes 32w .. 32w+31 (= rows), 8 columns per load
    for (int c = 0; c < N; c += 8) {
        uint32_t v[8];
        const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * N + c + j] = (int32_t)v[j];
    }
    if (tid == 0) cycles[0] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(N < 32 ? 32 : N));
}

template <int N>
int run(int K, int reps) {
    std::vector<int8_t> A(M * K), B(N * K);
    srand(7);
    for (auto &x : A) x = (int8_t)(rand() % 255 - 127);
    for (auto &x : B) x = (int8_t)(rand() % 255 - 127);
    int8_t *dA, *dB; int32_t *dD; long long *dc;
    cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    const int smem = (M + N) * K;
    cudaFuncSetAttribute(k_umma_i8<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_umma_i8<N><<<1, 128, smem>>>(dA, dB, K, reps, dD, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"N\":%d,\"err\":\"%s\"}\n", N, cudaGetErrorString(e)); return 1; }
    std::vector<int32_t> D(M * N);
    long long cyc;
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    long long bad = 0, first = -1;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            long long s = 0;
            for (int k = 0; k < K; ++k) s += (long long)A[i * K + k] * B[j * K + k];
            s *= reps;
            if ((int32_t)s != D[i * N + j]) { if (first < 0) first = i * N + j; ++bad; }
        }
    const double macs = (double)M * N * K * reps;
    printf("{\"N\":%d,\"K\":%d,\"reps\":%d,\"mismatches\":%lld,\"first_bad\":%lld,\"cycles\":%lld,\"mac_per_clk\":%.1f}\n",
           N, K, reps, bad, first, cyc, macs / (double)cyc);
    if (bad && first >= 0) {
        const int i = first / N, j = first % N;
        long long s = 0;
        for (int k = 0; k < K; ++k) s += (long long)A[i * K + k] * B[j * K + k];
        printf("  first bad (%d,%d): got %d want %lld\n", i, j, D[first], s * reps);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
    return bad != 0;
}

int main() {
    int fails = 0;
    fails += run<64>(64, 1);
    fails += run<128>(128, 1);
    fails += run<256>(256, 1);
    fails += run<128>(512, 64);     // rate: operands resident in smem
    fails += run<256>(256, 128);
    fails += run<64>(1024, 64);     // rate at N = 64 (the MC emulation's shape)
    return fails;
}
