// Blackwell tensor-core plumbing (tcgen05, sm_100a) for the exact integer
// contraction of the key switch: unsigned 8-bit operands in shared memory,
// 32-bit integer accumulators in Tensor Memory.
//
//   * operand layout: K-major, no swizzle ("interleaved" canonical layout):
//     8-row x 16-byte core matrices (rows 16 bytes apart, 128 contiguous
//     bytes); core matrices adjacent in K are LBO bytes apart, 8-row groups
//     SBO bytes apart;
//   * shared-memory matrix descriptor (64 bit): start >> 4 [0,14), LBO >> 4
//     [16,30), SBO >> 4 [32,46), version 1 [46,48), layout 0 = no swizzle;
//   * instruction descriptor (32 bit), kind::i8: D format S32 [4,6) = 2,
//     A / B format unsigned 8-bit (0), both K-major, N >> 3 [17,23),
//     M >> 4 [24,29);
//   * one elected thread issues tcgen05.mma; tcgen05.commit arrives on an
//     mbarrier when the issued MMAs have completed; the accumulator is read
//     with tcgen05.ld (warp w of a warpgroup sees lanes 32 (w % 4) .. + 31).
#pragma once
#include <cstdint>

namespace hefv {

__host__ __device__ constexpr uint64_t umma_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// K-major, 128-byte swizzle: rows of 128 bytes (K), 8-row atoms of 1024 bytes
// (1024-byte aligned), 16-byte chunk c of row r stored at chunk c ^ (r % 8);
// SBO = distance between 8-row atoms, LBO unused (1); layout type 2.
__host__ __device__ constexpr uint64_t umma_smem_desc_sw128(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// byte offset of (row r, byte k) in a K-major 128-byte-swizzled operand
__host__ __device__ constexpr uint32_t sw128_offset(uint32_t r, uint32_t k) {
  return (r >> 3) * 1024u + (r & 7u) * 128u + ((((k >> 4) ^ (r & 7u)) & 7u) << 4) + (k & 15u);
}

__host__ __device__ constexpr uint32_t umma_idesc_u8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[desc_a] x B[desc_b]^T, K = 32 bytes; accumulate != 0 adds.
__device__ __forceinline__ void umma_u8(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(
          tmem_d),
      "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
      : "memory");
}

// arrive on `mbar` once every tcgen05.mma issued so far by this thread is done
__device__ __forceinline__ void umma_commit(uint64_t* mbar) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   a)
               : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* smem_slot, uint32_t ncols) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(smem_slot);
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(a),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// shared-memory writes by threads -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32 lanes (one per thread of the warp) x 8 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr)
      : "memory");
}

}  // namespace hefv
