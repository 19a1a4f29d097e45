// Small device helpers shared by the kernel translation units.
#pragma once
#include "modarith.cuh"

namespace hefv {

__device__ __forceinline__ Mod32 make_mod(const Prime32Info& i) { return Mod32{i.p, 2 * i.p}; }
__device__ __forceinline__ Mod64 make_mod(const Prime64Info& i) { return Mod64{i.p, 2 * i.p}; }
__device__ __forceinline__ uint32_t reduce_any(uint32_t x, const Prime32Info& i) {
  return barrett62(x, i.p, i.mu);
}
__device__ __forceinline__ uint64_t reduce_any(uint64_t x, const Prime64Info& i) {
  return x >= i.p ? barrett64(x, i.p, i.mu) : x;
}

template <class M>
struct InfoOf;
template <>
struct InfoOf<Mod32> {
  typedef Prime32Info I;
};
template <>
struct InfoOf<Mod64> {
  typedef Prime64Info I;
};

// x canonical -> x * 2^32 mod p, canonical (Montgomery form)
__device__ __forceinline__ uint32_t mont_canon(uint32_t x, const Prime32Info& inf) {
  uint32_t r = mont_mul_lazy(x, inf.r2, inf.p, inf.pinv_neg);
  return r >= inf.p ? r - inf.p : r;
}

__device__ __forceinline__ int brev_n(int x, int logn) { return (int)(__brev((unsigned)x) >> (32 - logn)); }


// Streaming loads that do not allocate in L1 (keys, digits): L1 is kept for
// the twiddle tables that every CTA of the same prime re-reads.
__device__ __forceinline__ uint4 ld_stream_v4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Keys: keep in L2 (evict_last) -- every CTA of the same target prime re-reads them.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_key_v4(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// LOGE (log2 words per thread) used by the CTA-resident 32-bit transforms.
template <int LOGN>
struct Loge32 {
  static constexpr int v = LOGN >= 15 ? 5 : 4;
};

// ---- mbarrier + 1-D bulk copy (cp.async.bulk, the TMA engine's 1-D form) ---
__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}
// Issue (one thread): copy `bytes` (multiple of 16) from global `src` to shared
// `dst` (16-byte aligned), completing one phase of `mbar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* mbar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(d),
      "l"(src), "r"(bytes), "r"(m)
      : "memory");
}


}  // namespace hefv
