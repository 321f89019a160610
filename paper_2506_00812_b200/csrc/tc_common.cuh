// tcgen05 / TMA helpers shared by the tensor-core kernels (scan_tc.cu: the label-grouped scan;
// graph_build.cu: the per-label kNN self-join of the graph builder). Hand-written inline PTX for
// sm_100a: 2-D TMA tensor loads (tile and tile::gather4), shared-memory matrix descriptors for
// swizzled K-major operands, instruction descriptors, tcgen05.mma / commit / ld.
#pragma once
#include <cuda.h>
#include "common.cuh"

namespace vf {

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}
// 4 rows (global row ids r[0..3]) x one box width, landing as 4 consecutive swizzled rows
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, int x, const int32_t (&r)[4],
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, swizzle span `cw` bytes: 8-row core groups `8*cw`
// bytes apart (SBO); LBO is unused for swizzled K-major operands (encoded 1); version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, int cw) {
    const uint64_t layout = cw == 128 ? 2 : cw == 64 ? 4 : 6;
    return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)((8 * cw) >> 4) << 32) |
           ((uint64_t)1 << 46) | (layout << 61);
}

// Instruction descriptor, both operands K-major, M = 128 (the MMA's row count), N = n:
//   DT 0  kind::i8   u8 x u8 -> s32
//   DT 1  kind::tf32 tf32 x tf32 -> f32 (exact for the integer-valued data it is enabled for)
template <int DT>
__device__ __forceinline__ uint32_t idesc_of(int n) {
    const uint32_t fmt = DT == 0 ? (2u << 4) : ((1u << 4) | (2u << 7) | (2u << 10));
    return fmt | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int DT>
__device__ __forceinline__ void mma_issue(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    if constexpr (DT == 0)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
            ::"r"(tmem_d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
            ::"r"(tmem_d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
}

// ||v||^2 of one 4-byte word as an exact integer (u8: four bytes; f32: one integer-valued float)
template <int DT>
__device__ __forceinline__ uint32_t sq_word(uint32_t w, uint32_t acc) {
    if constexpr (DT == 0) return __dp4a(w, w, acc);
    const int v = __float2int_rn(__uint_as_float(w));
    return acc + (uint32_t)(v * v);
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Byte offset of 16-byte unit `u` of row `r` inside one swizzled K chunk (rows `cw` bytes apart):
// the hardware XORs address bits [4, 4+log2(cw/16)) with bits [7, ...) (Swizzle<b,4,3>).
__device__ __forceinline__ uint32_t swz(int r, int u, int cw) {
    const uint32_t o = (uint32_t)r * cw + (uint32_t)u * 16;
    const uint32_t m = (uint32_t)(cw / 16 - 1);
    return o ^ (((o >> 7) & m) << 4);
}


}  // namespace vf
