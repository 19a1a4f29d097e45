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
//   kind 10: VIADDMNMX (min(a, a - b), the butterflies' conditional subtract)
//   kind 11: LOP3 + add pair, kind 12: LOP3 + VIADDMNMX pair (ALU-pipe rates)
// Each thread runs 8 independent chains so the pipes, not latency, bound it.
#include "../../include/hefv.h"
#include "internal.h"
#include "kcommon.cuh"
#include "umma.cuh"

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
        } else if (KIND == 10) {
          a[i] = min(a[i], a[i] - b[i]);  // VIADDMNMX (the butterflies' conditional subtract)
        } else if (KIND == 11) {
          a[i] = (a[i] ^ b[i]) + b[i];  // LOP3 + add (counted as 1 op)
        } else if (KIND == 12) {
          const uint32_t v = a[i] ^ b[i];  // LOP3 + VIADDMNMX (counted as 1 op)
          a[i] = min(v, v - p2);
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

// tcgen05 int8 check: C (128 x 256, s32) = A (128 x K, u8) x B (256 x K, u8)^T
// with both operands K-major in the interleaved canonical layout; K = 32 * ks.
template <int M, bool SW>
__global__ void __launch_bounds__(128) k_probe_umma(const uint8_t* __restrict__ A,
                                                    const uint8_t* __restrict__ B,
                                                    int32_t* __restrict__ C, int ks) {
  constexpr int N = 256;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int K = 32 * ks;
  const uint32_t lbo = 128, sbo = SW ? 1024 : 128 * (K / 16);
  const int KR = SW ? 128 : K;  // bytes per stored row
  unsigned char* As = smraw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smraw) & 1023u)) & 1023u);
  unsigned char* Bs = As + M * KR;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  // canonical placement: (row r, byte k) -> (r/8) SBO + (k/16) LBO + (r%8) 16 + k%16
  for (int e = tid; e < M * KR; e += 128) {
    const int r = e / KR, k = e % KR;
    const unsigned char v = k < K ? A[r * K + k] : 0;
    As[SW ? sw128_offset(r, k) : (r / 8) * sbo + (k / 16) * lbo + (r % 8) * 16 + (k % 16)] = v;
  }
  for (int e = tid; e < N * KR; e += 128) {
    const int r = e / KR, k = e % KR;
    const unsigned char v = k < K ? B[r * K + k] : 0;
    Bs[SW ? sw128_offset(r, k) : (r / 8) * sbo + (k / 16) * lbo + (r % 8) * 16 + (k % 16)] = v;
  }
  if (tid == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) tmem_alloc(&tbase, N);
  fence_async_smem();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t td = tbase;
  if (tid == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(As);
    const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(Bs);
    const uint32_t idesc = umma_idesc_u8(M, N);
    for (int s = 0; s < ks; ++s) {
      if (SW)
        umma_u8(td, umma_smem_desc_sw128(a0 + 32 * s, sbo), umma_smem_desc_sw128(b0 + 32 * s, sbo),
                idesc, s > 0);
      else
        umma_u8(td, umma_smem_desc(a0 + 2 * lbo * s, lbo, sbo),
                umma_smem_desc(b0 + 2 * lbo * s, lbo, sbo), idesc, s > 0);
    }
    umma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tmem_fence_after();
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    tmem_ld8(td + ((uint32_t)(32 * w) << 16) + c0, v);
    tmem_wait_ld();
    // every TMEM lane is dumped (M = 64 shows where the 64 rows land)
    for (int j = 0; j < 8; ++j) C[(32 * w + lane) * N + c0 + j] = (int32_t)v[j];
  }
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(td, N);
}

// TMEM load-shape check: lane L, column c holds 1000 L + c (written with
// 32x32b stores); warp 0 then reads lanes 0.. with shape `shape` (0: 16x64b.x1,
// 1: 16x128b.x1, 2: 16x256b.x1) and dumps thread t's registers at out[t*4 + r].
__global__ void __launch_bounds__(128) k_probe_tmem_shape(int32_t* out, int shape) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  if (w == 0) tmem_alloc(&tbase, 32);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t lrow = (uint32_t)(32 * w + lane);
  for (int c = 0; c < 32; ++c) {
    const uint32_t v = lrow * 1000u + (uint32_t)c;
    const uint32_t ta = tbase + ((uint32_t)(32 * w) << 16) + (uint32_t)c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta), "r"(v) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (w == 0) {
    uint32_t r[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
    if (shape == 0) {
      asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(tbase) : "memory");
    } else if (shape == 1) {
      asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(tbase) : "memory");
    } else {
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tbase) : "memory");
    }
    tmem_wait_ld();
    for (int q = 0; q < 4; ++q) out[lane * 4 + q] = (int32_t)r[q];
  }
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, 32);
}

// tcgen05 MMA latency / throughput (development aid): one CTA, operands in
// shared memory (contents irrelevant), `chain` MMAs (M = 64, N = 128, K = 32,
// u8) into one accumulator per commit; mode 0: wait after every commit
// (latency), mode 1: `depth` commits in flight over `depth` accumulators.
// out[0] = clock64 cycles for `reps` commits.
__global__ void __launch_bounds__(128) k_probe_umma_lat(int64_t* out, int reps, int chain, int depth,
                                                        int sw, int M, int N) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[8];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid >> 5;
  unsigned char* base = smraw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smraw) & 1023u)) & 1023u);
  for (int e = tid; e < 128 * 128 + 256 * 128; e += 128) base[e] = (unsigned char)e;
  if (tid == 0) {
    for (int q = 0; q < 8; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) tmem_alloc(&tbase, 512);
  fence_async_smem();
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  if (tid == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(base);
    const uint32_t b0 = a0 + 128 * 128;
    const uint32_t idesc = umma_idesc_u8(M, N);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int slot = r % depth;
      if (r >= depth) mbar_wait(&bars[slot], (uint32_t)(((r - depth) / depth) & 1));
      for (int c = 0; c < chain; ++c) {
        if (sw)
          umma_u8(tbase + (uint32_t)slot * (uint32_t)N, umma_smem_desc_sw128(a0 + 32 * (c % 3), 1024),
                  umma_smem_desc_sw128(b0 + 32 * (c % 3), 1024), idesc, c > 0);
        else
          umma_u8(tbase + (uint32_t)slot * (uint32_t)N, umma_smem_desc(a0 + 256 * (c % 3), 128, 768),
                  umma_smem_desc(b0 + 256 * (c % 3), 128, 768), idesc, c > 0);
      }
      umma_commit(&bars[slot]);
    }
    for (int r = (reps > depth ? reps - depth : 0); r < reps; ++r)
      mbar_wait(&bars[r % depth], (uint32_t)((r / depth) & 1));
    out[0] = clock64() - t0;
  }
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, 512);
}

}  // namespace hefv

using namespace hefv;

extern "C" int hefv_probe_umma_lat(int64_t* out, int32_t reps, int32_t chain, int32_t depth,
                                   void* stream) {
  // depth: +-(d + 4 * shape), shape 0: M64 N128, 1: M128 N128, 2: M128 N256, 3: M64 N256
  const int sw = depth < 0;
  if (sw) depth = -depth;
  const int shape = (depth - 1) / 4;
  depth = (depth - 1) % 4 + 1;
  const int M = (shape == 1 || shape == 2) ? 128 : 64, N = (shape >= 2) ? 256 : 128;
  if (depth * N > 512) depth = 512 / N;
  const size_t smem = 128 * 128 + 256 * 128 + 1024;
  if (cudaFuncSetAttribute(k_probe_umma_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return fail("hefv_probe_umma_lat: smem attribute");
  k_probe_umma_lat<<<1, 128, smem, as_stream(stream)>>>(out, reps, chain, depth, sw, M, N);
  HEFV_LAUNCH_CHECK("k_probe_umma_lat");
  return 0;
}

extern "C" int hefv_probe_tmem_shape(int32_t* out, int32_t shape, void* stream) {
  k_probe_tmem_shape<<<1, 128, 0, as_stream(stream)>>>(out, shape);
  HEFV_LAUNCH_CHECK("k_probe_tmem_shape");
  return 0;
}

extern "C" int hefv_probe_umma(const uint8_t* A, const uint8_t* B, int32_t* C, int32_t ks,
                               void* stream) {
  // ks > 0: M = 128; ks < 0: M = 64 (A has 64 rows, C still dumps 128 lanes);
  // |ks| >= 8: 128-byte swizzled operands with |ks| - 8 k-steps
  const bool m64 = ks < 0;
  if (m64) ks = -ks;
  const bool sw = ks >= 8;
  if (sw) ks -= 8;
  if (ks < 1 || ks > 4) return fail("hefv_probe_umma: |ks| must be 1..4 (+8 swizzled)");
  const size_t smem = (size_t)(128 + 256) * 128 + 1024;
  auto kern = m64 ? (sw ? k_probe_umma<64, true> : k_probe_umma<64, false>)
                  : (sw ? k_probe_umma<128, true> : k_probe_umma<128, false>);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return fail("hefv_probe_umma: smem attribute");
  kern<<<1, 128, smem, as_stream(stream)>>>(A, B, C, ks);
  HEFV_LAUNCH_CHECK("k_probe_umma");
  return 0;
}

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
    case 10:
      k_probe<10><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 11:
      k_probe<11><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    case 12:
      k_probe<12><<<blocks, 256, 0, st>>>(out, iters, 7u);
      break;
    default:
      return fail("hefv_probe_int: unknown kind");
  }
  HEFV_LAUNCH_CHECK("k_probe");
  return 0;
}
