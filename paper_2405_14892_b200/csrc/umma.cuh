// tcgen05 / cluster helpers shared by the int8 tensor-core kernels (kernels_mc_oz.cu: MC validation,
// kernels_sov_oz.cu: the SOV GEMM). No-swizzle K-major operands in the canonical core-matrix order.
#pragma once
#include "common.cuh"

namespace mvn {

// Shared-memory matrix descriptor of a K-major no-swizzle operand: SBO (next 8-row group) = 256 B,
// LBO (next 16-byte K group) = 128 B, version 1.
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
    // SBO (next 8-row group) = 256 B, LBO (next 16-byte K group) = 128 B, version 1, no swizzle
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}

// Byte offset of element (row, k) (k < 32) inside one slice of a [rows x 32] K-major operand in
// the canonical core-matrix order [row / 8][k / 16][row % 8][k % 16].
__device__ __forceinline__ int oz_core(int row, int k) { return ((row >> 3) << 8) + ((k >> 4) << 7) + ((row & 7) << 4) + (k & 15); }

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_peer(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAITC_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAITC_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// kind::i8 instruction descriptor: D s32, A/B signed, K-major, M = 128, N = n.
constexpr uint32_t i8_idesc(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

}  // namespace mvn
