// Device primitives shared by the libmvn kernels (sm_100a only).
//  - fp64 tensor-core MMA: mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4. tcgen05 has no f64 kind on
//    sm_100a (ptxas rejects .kind::f64), so warp-level DMMA with register operands is the fp64
//    tensor path; measured 37.07 TFLOP/s = the chip's fp64 peak (profiles/r01_fp64_calibration.md).
//  - cp.async 16-byte global->shared copies (LDGSTS) for multi-stage operand pipelines.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "mvn_internal.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libmvn is built for sm_100a (B200) only"
#endif

namespace mvn {

__host__ __device__ inline int64_t tile_offset(int64_t i, int64_t j) {
    return ((i * (i + 1)) / 2 + j) * (int64_t)kTile * kTile;
}

// C(8x8) += A(8x4, row) * B(4x8, col). Fragment ownership (lane l):
//   a = A[l/4][l%4], b = B[l%4][l/4], c = {C[l/4][2(l%4)], C[l/4][2(l%4)+1]}
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- named barriers, mbarriers and TMA bulk copies (SASS: BAR, SYNCS.*, UBLKCP)
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

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
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// TMA-engine bulk copy global -> shared, completion counted on an mbarrier (SASS UBLKCP).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// Arrive on an mbarrier when all of this thread's prior cp.async copies have landed (the pending
// count is raised now and dropped at completion, so the phase cannot complete before them).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Bulk prefetch of a global range into L2 (no shared-memory destination).
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace mvn
