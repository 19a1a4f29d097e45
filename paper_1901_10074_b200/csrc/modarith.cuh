// Modular arithmetic primitives for the RNS/FV hot path (sm_100a).
//
// Two word sizes:
//   * Mod32 -- the FV q / auxiliary primes (30-bit, 2^28 < p < 2^30, see
//     fv.py:60-64 and fv.py:89-95 of the reference: `find_ntt_primes(count,
//     30, 2n)`).  Twiddle products use Shoup's trick with a 32-bit companion
//     (the same constant family as ntt.py:166-170), key products use
//     Montgomery REDC so the switch keys stay at one word per coefficient.
//   * Mod64 -- the plaintext modulus t (18..53 bits at the shipped profiles)
//     and the 50-62-bit primes of the kernel microbench (config 4).  Shoup
//     with a 64-bit companion; requires p < 2^62 so lazy values < 4p fit.
//
// All butterflies are Harvey-style lazy: forward (Cooley-Tukey) keeps
// values in [0, 4p), inverse (Gentleman-Sande) in [0, 2p).  Results leave a
// kernel only after the final correction to the canonical range [0, p), so
// every limb that reaches HBM is bit-identical to the reference's
// canonical residues.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hefv {

// ptxas balances the FMA and ALU pipes by instruction COUNT and lowers plain
// 32-bit adds to IMAD.IADD to do so; on sm_100a IMAD.HI / IMAD.WIDE issue at
// half rate, so a forward butterfly loads the FMA pipe with 11 cycles against
// the ALU's 8 (ncu, profiles/r02).  alu_add keeps an add on the ALU pipe:
// min(a + b, 0xffffffff) with the constant opaque to the compiler is one
// VIADDMNMX, which has no FMA-pipe form.  Measured (B200): 2^14 forward
// +3.6 %; the inverse (-1.5 %) and the 2^12 forward (-2.4 %) lose, so only
// the 2^14 forwards use the *A types below.
__device__ __forceinline__ uint32_t opaque_ones() {
  uint32_t v = 0xffffffffu;
  asm volatile("" : "+r"(v));
  return v;
}
__device__ __forceinline__ uint32_t alu_add(uint32_t a, uint32_t b, uint32_t ones) {
  return min(a + b, ones);
}

// ---------------------------------------------------------------- 32-bit
struct Mod32 {
  typedef uint32_t T;
  typedef uint2 Tw;  // (w, floor(w * 2^32 / p))
  uint32_t p, p2;

  __device__ __forceinline__ static uint32_t mul_shoup(uint32_t x, uint32_t w, uint32_t wsh,
                                                       uint32_t p) {
    uint32_t q = __umulhi(x, wsh);
    return x * w - q * p;  // in [0, 2p) for any x < 2^32
  }
  __device__ __forceinline__ uint32_t sub2p(uint32_t x) const { return min(x, x - p2); }
  __device__ __forceinline__ uint32_t subp(uint32_t x) const { return min(x, x - p); }
  // canonical from [0, 4p)
  __device__ __forceinline__ uint32_t canon4(uint32_t x) const { return subp(sub2p(x)); }
  __device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, Tw w) const {
    uint32_t a = sub2p(x);
    uint32_t t = mul_shoup(y, w.x, w.y, p);
    x = a + t;
    y = a - t + p2;
  }
  __device__ __forceinline__ void gs(uint32_t& x, uint32_t& y, Tw w) const {
    uint32_t a = x, b = y;
    x = sub2p(a + b);
    y = mul_shoup(a - b + p2, w.x, w.y, p);
  }
  // last inverse stage with N^{-1} merged: x' = (a+b) n^-1, y' = (a-b) w n^-1
  __device__ __forceinline__ void gs_last(uint32_t& x, uint32_t& y, Tw ninv, Tw wn) const {
    uint32_t a = x, b = y;
    x = mul_shoup(a + b, ninv.x, ninv.y, p);
    y = mul_shoup(a - b + p2, wn.x, wn.y, p);
  }
};

// Word-sized prime with single-word Montgomery-form twiddles (w * 2^32 mod p):
// half the twiddle bytes of the Shoup pair, so a full forward table of a
// 2^14-point transform fits in shared memory next to the data tile.
struct Mod32M {
  typedef uint32_t T;
  typedef uint32_t Tw;
  uint32_t p, p2, pinv;  // pinv = p^{-1} mod 2^32

  // y * w * 2^-32 mod p in (0, 2p) for y < 2^32, w < p
  __device__ __forceinline__ uint32_t mul(uint32_t y, uint32_t w) const {
    const uint64_t t = (uint64_t)y * w;
    const uint32_t m = (uint32_t)t * pinv;
    return (uint32_t)(t >> 32) - __umulhi(m, p) + p;
  }
  __device__ __forceinline__ uint32_t sub2p(uint32_t x) const { return min(x, x - p2); }
  __device__ __forceinline__ uint32_t subp(uint32_t x) const { return min(x, x - p); }
  __device__ __forceinline__ uint32_t canon4(uint32_t x) const { return subp(sub2p(x)); }
  __device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, Tw w) const {
    uint32_t a = sub2p(x);
    uint32_t t = mul(y, w);
    x = a + t;
    y = a - t + p2;
  }
  // Gentleman-Sande, inputs < 2p -> outputs < 2p (as Mod32::gs)
  __device__ __forceinline__ void gs(uint32_t& x, uint32_t& y, Tw w) const {
    uint32_t a = x, b = y;
    x = sub2p(a + b);
    y = mul(a - b + p2, w);
  }
  // last inverse stage with N^{-1} merged (Montgomery-form ninv, wn)
  __device__ __forceinline__ void gs_last(uint32_t& x, uint32_t& y, Tw ninv, Tw wn) const {
    uint32_t a = x, b = y;
    x = mul(a + b, ninv);
    y = mul(a - b + p2, wn);
  }
};

// Forward-butterfly variants with the sum forced onto the ALU pipe (alu_add).
struct Mod32A : Mod32 {
  uint32_t ones;
  __device__ __forceinline__ explicit Mod32A(uint32_t p_) : Mod32{p_, 2 * p_}, ones(opaque_ones()) {}
  __device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, Tw w) const {
    uint32_t a = sub2p(x);
    uint32_t t = mul_shoup(y, w.x, w.y, p);
    x = alu_add(a, t, ones);
    y = a - t + p2;
  }
};
struct Mod32MA : Mod32M {
  uint32_t ones;
  __device__ __forceinline__ Mod32MA(uint32_t p_, uint32_t pinv_, uint32_t ones_)
      : Mod32M{p_, 2 * p_, pinv_}, ones(ones_) {}
  __device__ __forceinline__ void ct(uint32_t& x, uint32_t& y, Tw w) const {
    uint32_t a = sub2p(x);
    uint32_t t = mul(y, w);
    x = alu_add(a, t, ones);
    y = a - t + p2;
  }
};

// Montgomery REDC for a*b with b < p and a < 2^32: returns a*b*2^-32 mod p in [0, 2p).
__device__ __forceinline__ uint32_t mont_mul_lazy(uint32_t a, uint32_t b, uint32_t p,
                                                  uint32_t pinv_neg) {
  uint64_t t = (uint64_t)a * b;
  uint32_t lo = (uint32_t)t;
  uint32_t m = lo * pinv_neg;
  uint32_t h = __umulhi(m, p);
  return (uint32_t)(t >> 32) + h + (lo != 0u);
}

// ---------------------------------------------------------------- 64-bit
struct Mod64 {
  typedef uint64_t T;
  typedef ulonglong2 Tw;  // (w, floor(w * 2^64 / p))
  uint64_t p, p2;

  __device__ __forceinline__ static uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t wsh,
                                                       uint64_t p) {
    uint64_t q = __umul64hi(x, wsh);
    return x * w - q * p;  // in [0, 2p)
  }
  __device__ __forceinline__ uint64_t sub2p(uint64_t x) const { return x >= p2 ? x - p2 : x; }
  __device__ __forceinline__ uint64_t subp(uint64_t x) const { return x >= p ? x - p : x; }
  __device__ __forceinline__ uint64_t canon4(uint64_t x) const { return subp(sub2p(x)); }
  __device__ __forceinline__ void ct(uint64_t& x, uint64_t& y, Tw w) const {
    uint64_t a = sub2p(x);
    uint64_t t = mul_shoup(y, w.x, w.y, p);
    x = a + t;
    y = a - t + p2;
  }
  __device__ __forceinline__ void gs(uint64_t& x, uint64_t& y, Tw w) const {
    uint64_t a = x, b = y;
    x = sub2p(a + b);
    y = mul_shoup(a - b + p2, w.x, w.y, p);
  }
  __device__ __forceinline__ void gs_last(uint64_t& x, uint64_t& y, Tw ninv, Tw wn) const {
    uint64_t a = x, b = y;
    x = mul_shoup(a + b, ninv.x, ninv.y, p);
    y = mul_shoup(a - b + p2, wn.x, wn.y, p);
  }
};

// Full 64x64 -> mod p product for p < 2^62 (variable x variable); used off the
// transform path (pointwise products of 64-bit residues).
__device__ __forceinline__ uint64_t mulmod64(uint64_t a, uint64_t b, uint64_t p) {
  unsigned __int128 t = (unsigned __int128)a * b;
  return (uint64_t)(t % p);
}

// Barrett reduction of x < 2^62 by a 30-bit prime with mu = floor(2^64 / p).
__device__ __forceinline__ uint32_t barrett62(uint64_t x, uint32_t p, uint64_t mu) {
  uint64_t q = __umul64hi(x, mu);
  uint64_t r = x - q * p;
  return (uint32_t)(r >= p ? r - p : r);
}

// Per-prime constants (one record per 32-bit prime of a context).
struct Prime32Info {
  uint32_t p;
  uint32_t pinv_neg;  // -p^{-1} mod 2^32
  uint32_t r2;        // 2^64 mod p (to enter Montgomery form)
  uint32_t pad;
  uint64_t mu;        // floor(2^64 / p)
  uint2 ninv;         // (N^{-1}, shoup)
  uint2 wn;           // (psi_inv_rev[1] * N^{-1}, shoup)
  uint32_t pinv;      // p^{-1} mod 2^32
  uint32_t pad2;
};

struct Prime64Info {
  uint64_t p;
  ulonglong2 ninv;
  ulonglong2 wn;
  uint64_t pinv_neg;  // -p^{-1} mod 2^64 (Montgomery)
  uint64_t r2;        // 2^128 mod p
  uint64_t mu;        // floor(2^64 / p) (Barrett)
};

// x mod p for any x < 2^64 and 2 <= p < 2^62 without a division call:
// q = hi(x mu) lies within 2 of floor(x / p), so x - q p < 3p.
__device__ __forceinline__ uint64_t barrett64(uint64_t x, uint64_t p, uint64_t mu) {
  uint64_t r = x - __umul64hi(x, mu) * p;
  r = r >= p ? r - p : r;
  return r >= p ? r - p : r;
}

// 64-bit Montgomery REDC of a*b (a < 2^64, b < p < 2^62): a*b*2^-64 mod p in [0, 2p).
__device__ __forceinline__ uint64_t mont_mul64_lazy(uint64_t a, uint64_t b, uint64_t p,
                                                    uint64_t pinv_neg) {
  const uint64_t lo = a * b;
  const uint64_t hi = __umul64hi(a, b);
  const uint64_t m = lo * pinv_neg;
  return hi + __umul64hi(m, p) + (lo != 0ull);
}

}  // namespace hefv
