// Integer-pipe peak probe.  MEASURED_PEAKS.json only carries HBM and bf16
// figures; the NTT / key-switch roofline needs the integer multiply rates of
// this part, so this kernel measures them (ops per second over the whole
// GPU) for the instruction forms the transforms use:
//   kind 0: IMAD      (32-bit multiply-add, low word)
//   kind 1: IMAD.HI   (__umulhi)
//   kind 2: IMAD.WIDE (32x32 -> 64-bit product)
//   kind 3: IADD3     (ALU pipe reference)
//   kind 4: one lazy Shoup Cooley-Tukey butterfly (counted as 1 op)
//   kind 5: one lazy 64-bit Shoup butterfly (p < 2^62; counted as 1 op)
//   kind 6: mad.wide.u32 into a 64-bit running sum whose bits feed the next
//           multiplier (a dependent chain: the product cannot be hoisted)
//   kind 7: DFMA (fp64 fused multiply-add)
//   kind 8: the kind-4 butterfly with its quotient on the FP64 pipe
//   kind 9: kinds 4 and 8 interleaved (half the chains each)
// Each thread runs 8 independent chains so the pipes, not latency, bound it.
#include "../../include/hefv.h"
#include "internal.h"

namespace hefv {

__global__ void __launch_bounds__(256) k_probe64(uint32_t* out, int iters, uint32_t seed) {
  uint64_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = (uint64_t)(seed * (threadIdx.x + 1) + i) * 0x9e3779b97f4a7c15ull >> 3;
    b[i] = ((uint64_t)(seed ^ (blockIdx.x * 131u + i)) * 0xbf58476d1ce4e5b9ull) >> 3;
  }
  const uint64_t p = 4611686018427322369ull, p2 = 2 * p;  // 2^62 - 2^16 + 1 (prime)
  const uint64_t w = 1234567890123456789ull % p, wsh = (uint64_t)(((unsigned __int128)w << 64) / p);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint64_t x = a[i] >= p2 ? a[i] - p2 : a[i];
        const uint64_t q = __umul64hi(b[i], wsh);
        const uint64_t t = b[i] * w - q * p;
        a[i] = x + t;
        b[i] = x - t + p2;
      }
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i] ^ b[i];
  if (s == 0x12345678ull) out[0] = (uint32_t)s;
}

template <int KIND>
__global__ void __launch_bounds__(256) k_probe(uint32_t* out, int iters, uint32_t seed) {
  uint32_t a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
    b[i] = (seed ^ (blockIdx.x * 131u + i)) | 1u;
  }
  const uint32_t p = 1073692673u, p2 = 2u * p;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (KIND == 0) {
          a[i] = a[i] * b[i] + 0x1234567u;
        } else if (KIND == 1) {
          a[i] = __umulhi(a[i], b[i]) ^ b[i];
        } else if (KIND == 2) {
          const uint64_t t = (uint64_t)a[i] * b[i];
          a[i] = (uint32_t)t ^ (uint32_t)(t >> 32);
        } else if (KIND == 3) {
          a[i] = a[i] + b[i] + 0x777u;
        } else if (KIND == 8 || (KIND == 9 && (i & 1))) {
          // the same butterfly with the Shoup quotient taken on the FP64
          // pipe: q = rint(y * w / p) from y as an exact double (magic-
          // number conversion), t = y w - q p + p in [0, 2p)
          const uint32_t w = 123456789u;
          const double wf = 123456789.0 / 1073692673.0;
          uint32_t x = min(a[i], a[i] - p2);
          const double yd = __hiloint2double(0x43300000, b[i]) - 4503599627370496.0;
          const uint32_t q = (uint32_t)__double2loint(fma(yd, wf, 6755399441055744.0));
          const uint32_t t = b[i] * w + p - q * p;
          a[i] = x + t;
          b[i] = x - t + p2;
        } else {
          // x = a[i], y = b[i] butterfly with twiddle (w, wsh)
          const uint32_t w = 123456789u, wsh = 493903u;
          uint32_t x = min(a[i], a[i] - p2);
          const uint32_t q = __umulhi(b[i], wsh);
          const uint32_t t = b[i] * w - q * p;
          a[i] = x + t;
          b[i] = x - t + p2;
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= a[i] ^ b[i];
  if (s == 0x12345678u) out[0] = s;  // keep the work alive
}

__global__ void __launch_bounds__(256) k_probe_madwide(uint32_t* out, int iters, uint32_t seed) {
  uint64_t acc[8];
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc[i] = seed + i;
    a[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
  }
  const uint32_t b = seed | 0x10001u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // multiplier taken from the running sum: no product can be hoisted
        const uint32_t m = (uint32_t)(acc[i] >> 7) | b;
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"(a[i]), "r"(m));
      }
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= acc[i];
  if (s == 0x12345678ull) out[0] = (uint32_t)s;
}

__global__ void __launch_bounds__(256) k_probe_dfma(uint32_t* out, int iters, uint32_t seed) {
  double acc[8];
  const double b = 1.0000001 + seed * 1e-9;
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc[i] = i;
    a[i] = 0.5 + threadIdx.x * 1e-6 + i;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(a[i], b, acc[i]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = 1u;
}

}  // namespace hefv

using namespace hefv;

// ops executed = blocks * 256 threads * iters * 16 * 8
extern "C" int hefv_probe_int(int32_t kind, int32_t blocks, int32_t iters, uint32_t* out,
                              void* stream) {
  cudaStream_t st = as_stream(stream);
  switch (kind) {
    case 0:
      k_probe<0><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 1:
      k_probe<1><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 2:
      k_probe<2><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 3:
      k_probe<3><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 4:
      k_probe<4><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 5:
      k_probe64<<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 6:
      k_probe_madwide<<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 7:
      k_probe_dfma<<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 8:
      k_probe<8><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 9:
      k_probe<9><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    default:
      return fail("hefv_probe_int: unknown kind");
  }
  HEFV_LAUNCH_CHECK("k_probe");
  return 0;
}
