// Micro-benchmark (tooling, not product): throughput of TMA bulk copies (cp.async.bulk) of
// different sizes into a 4-stage shared-memory ring, one producer lane per CTA, consumers only
// wait + release. Compares with per-thread cp.async 16 B. Prints GB/s for the whole GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

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
    asm volatile("{\n .reg .pred p;\nWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

constexpr int STAGES = 4, STAGE_BYTES = 32768;

// each stage = STAGE_BYTES moved as `ncopy` copies of STAGE_BYTES/ncopy bytes, issued by the 32 lanes
__global__ void k_tma(const char *src, size_t span, int iters, int ncopy, double *sink) {
    extern __shared__ __align__(128) char sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + STAGES * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned csz = STAGE_BYTES / ncopy;
    if (warp == 8) {
        for (int q = 0; q < iters; ++q) {
            const int st = q % STAGES;
            mbar_wait(&empty[st], ((q / STAGES) & 1) ^ 1);
            if (lane == 0) mbar_arrive_expect_tx(&full[st], STAGE_BYTES);
            __syncwarp();
            size_t off = ((size_t)(blockIdx.x * (size_t)iters + q) * STAGE_BYTES) % span;
            for (int c = lane; c < ncopy; c += 32) bulk_g2s(sm + st * STAGE_BYTES + c * csz, src + off + c * csz, csz, &full[st]);
        }
    } else {
        double acc = 0;
        for (int q = 0; q < iters; ++q) {
            const int st = q % STAGES;
            mbar_wait(&full[st], (q / STAGES) & 1);
            acc += reinterpret_cast<const double *>(sm + st * STAGE_BYTES)[threadIdx.x];
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (acc == 1.2345) sink[0] = acc;
    }
}

__global__ void k_cpasync(const char *src, size_t span, int iters, double *sink) {
    extern __shared__ __align__(128) char sm[];
    double acc = 0;
    for (int q = 0; q < iters; ++q) {
        const int st = q % STAGES;
        size_t off = ((size_t)(blockIdx.x * (size_t)iters + q) * STAGE_BYTES) % span;
        for (int e = threadIdx.x; e < STAGE_BYTES / 16; e += 256) {
            unsigned s = smem_u32(sm + st * STAGE_BYTES + e * 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + off + e * 16));
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 2;\n" ::);
        __syncthreads();
        acc += reinterpret_cast<const double *>(sm + ((q + 2) % STAGES) * STAGE_BYTES)[threadIdx.x];
        __syncthreads();
    }
    if (acc == 1.2345) sink[0] = acc;
}

int main() {
    size_t span = (size_t)4 << 30;  // 4 GB > L2
    char *src; double *sink;
    cudaMalloc(&src, span + (1 << 20));
    cudaMemset(src, 0, span);
    cudaMalloc(&sink, 8);
    int smem = STAGES * STAGE_BYTES + 128;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2000, grid = 148;
    for (size_t sp : {span, (size_t)(64 << 20)}) {
        for (int ncopy : {1, 2, 8, 16, 32, 64}) {
            k_tma<<<grid, 288, smem>>>(src, sp, 50, ncopy, sink);
            cudaEventRecord(e0);
            k_tma<<<grid, 288, smem>>>(src, sp, iters, ncopy, sink);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"kind\":\"tma\",\"span_MB\":%zu,\"copies_per_32KB\":%d,\"copy_bytes\":%d,\"GBs\":%.1f}\n", sp >> 20, ncopy,
                   STAGE_BYTES / ncopy, (double)grid * iters * STAGE_BYTES / ms / 1e6);
        }
        k_cpasync<<<grid, 256, smem>>>(src, sp, 50, sink);
        cudaEventRecord(e0);
        k_cpasync<<<grid, 256, smem>>>(src, sp, iters, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"kind\":\"cp.async16\",\"span_MB\":%zu,\"GBs\":%.1f}\n", sp >> 20, (double)grid * iters * STAGE_BYTES / ms / 1e6);
    }
    printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
