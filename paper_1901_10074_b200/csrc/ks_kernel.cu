// Fused RNS-limb key switch (K4).  Replaces _keyswitch_apply (reference
// fv.py:205-217):
//     for each target prime j:
//         digits = NTT_j(c mod p_j)            (k forward NTTs)
//         acc0   = sum_i digits_i * body[j]_i  (MAC over k digits)
//         acc1   = sum_i digits_i * mask[j]_i
//         (d0_j, d1_j) = iNTT_j(acc0, acc1)
// One CTA owns one (target prime j, ciphertext b) pair for the whole
// pipeline: each digit is loaded coalesced from L2/HBM, transformed in
// registers + one shared tile, multiplied into register-resident
// accumulators (Montgomery REDC against the Montgomery-form key, lazy in
// [0, 2p)), and the two accumulators are inverse-transformed and written
// once, fused with the caller's epilogue additions (sigma(c0) for a
// rotation hop, the running sum for all_sum, t0/t1 for relinearisation).
// Nothing but the final (d0, d1) + addends ever reaches HBM.
//
// Digits enter the transform unreduced: c_i < p_i < 2^30 < 4 p_j, which the
// lazy Cooley-Tukey butterflies accept (ctx setup checks p_j > 2^28).
#include "../../include/hefv.h"
#include "internal.h"
#include "kcommon.cuh"
#include "ntt.cuh"

namespace hefv {

#ifndef HEFV_KS_LOGE14
#define HEFV_KS_LOGE14 4
#endif
template <int LOGN>
struct KsLoge {
  static constexpr int v = LOGN >= 15 ? 5 : (LOGN == 14 ? HEFV_KS_LOGE14 : 4);
};

// Ciphertexts handled per CTA: the forward twiddle table of the CTA's prime
// is staged in shared memory once and reused for CH * k digit transforms.
#ifndef HEFV_KS_CTS
#define HEFV_KS_CTS 4
#endif
constexpr int KS_CTS_PER_CTA = HEFV_KS_CTS;

// Shared memory: Montgomery-form forward twiddles of prime j (N words), the
// padded exchange tile, and the mask accumulator acc1 (N words, laid out
// [register e][thread] so every thread touches its own conflict-free words).
// The body accumulator acc0 and the digit being transformed stay in
// registers (2 E words per thread).
template <int LOGN, int LOGE>
__global__ void __launch_bounds__(Geo<LOGN, LOGE>::NT,
                                  Geo<LOGN, LOGE>::NT >= 1024 ? 1 : 1024 / Geo<LOGN, LOGE>::NT)
    k_keyswitch(const uint32_t* __restrict__ kbody, const uint32_t* __restrict__ kmask,
                const uint32_t* __restrict__ digits, int64_t dig_stride, uint32_t* out0,
                uint32_t* out1, int64_t out_stride, const int32_t* __restrict__ slot,
                const uint32_t* __restrict__ adA0, const uint32_t* __restrict__ adA1,
                int64_t adA_stride, const uint32_t* adB0, const uint32_t* adB1, int64_t adB_stride,
                int64_t B, int k, const uint2* __restrict__ tw_all,
                const uint2* __restrict__ itw_all, const Prime32Info* __restrict__ info) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int E = G_::E;
  constexpr int NT = G_::NT;
  constexpr int N = G_::N;
  constexpr int R = G_::RLAST;
  extern __shared__ __align__(16) unsigned char smraw[];
  // Shoup twiddles of the full passes ([1, 2^(LOGN-RLAST))) in shared
  // memory; the last pass reads its N - 2^(LOGN-RLAST) entries through L1.
  constexpr int NTW = 1 << (LOGN - R);
  uint2* tws = reinterpret_cast<uint2*>(smraw);
  uint32_t* sm = reinterpret_cast<uint32_t*>(tws + NTW);  // exchange tile
  uint32_t* acc1s = sm + ((spad_size(N) + 3) & ~3);      // mask accumulator (16B aligned)
  const int j = blockIdx.x;
  const int tid = threadIdx.x;
  const Prime32Info inf = info[j];
  const Mod32 md{inf.p, 2 * inf.p};
  const uint2* twg = tw_all + (size_t)j * N;
  {
    const uint4* src = reinterpret_cast<const uint4*>(twg);
    uint4* dst = reinterpret_cast<uint4*>(tws);
    for (int i = tid; i < NTW / 2; i += NT) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const uint64_t kpol = l2_policy_evict_last();
  const uint2* itw = itw_all + (size_t)j * N;
  const int64_t bbeg = (int64_t)blockIdx.y * KS_CTS_PER_CTA;
  const int64_t bend = min(B, bbeg + KS_CTS_PER_CTA);

  // mask accumulator in shared memory as [E/4][NT] 16-byte chunks: thread
  // tid's chunk q sits at q * NT + tid, so a quarter-warp's 128-bit accesses
  // cover 128 consecutive bytes (conflict-free)
  uint4* acc1v = reinterpret_cast<uint4*>(acc1s);
  const Mod32M mm{inf.p, 2 * inf.p, inf.pinv};
  for (int64_t b = bbeg; b < bend; ++b) {
    const uint32_t* dig = digits + b * dig_stride;
    uint32_t acc0[E], x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc0[e] = 0u;
#pragma unroll
    for (int q = 0; q < E / 4; ++q) acc1v[q * NT + tid] = make_uint4(0u, 0u, 0u, 0u);

    for (int i = 0; i < k; ++i) {
      {
        const uint32_t* src = dig + (size_t)i * N;
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = ld_stream(src + tid + e * NT);
      }
      cta_fwd<LOGN, LOGE, Mod32>(md, x, sm, tws, twg, NoHook(), LOGN - R);
      const size_t koff = ((size_t)j * k + i) * N + row_index<LOGN, LOGE>(tid, 0);
      const uint4* kb = reinterpret_cast<const uint4*>(kbody + koff);
      const uint4* km = reinterpret_cast<const uint4*>(kmask + koff);
#pragma unroll
      for (int q = 0; q < E / 4; ++q) {
        const uint4 wb = ld_key_v4(kb + q, kpol);
        const uint4 wm = ld_key_v4(km + q, kpol);
        uint4 a1 = acc1v[q * NT + tid];
        const uint32_t kbv[4] = {wb.x, wb.y, wb.z, wb.w};
        const uint32_t kmv[4] = {wm.x, wm.y, wm.z, wm.w};
        uint32_t a1v[4] = {a1.x, a1.y, a1.z, a1.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int e = q * 4 + r;
          acc0[e] = md.sub2p(acc0[e] + mm.mul(x[e], kbv[r]));
          a1v[r] = md.sub2p(a1v[r] + mm.mul(x[e], kmv[r]));
        }
        acc1v[q * NT + tid] = make_uint4(a1v[0], a1v[1], a1v[2], a1v[3]);
      }
    }

    const int64_t s = slot ? (int64_t)slot[b] : b;
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      if (part == 1) {
#pragma unroll
        for (int q = 0; q < E / 4; ++q) {
          const uint4 a1 = acc1v[q * NT + tid];
          acc0[4 * q] = a1.x;
          acc0[4 * q + 1] = a1.y;
          acc0[4 * q + 2] = a1.z;
          acc0[4 * q + 3] = a1.w;
        }
      }
      cta_inv<LOGN, LOGE, Mod32>(md, acc0, sm, itw, inf.ninv, inf.wn);
      uint32_t* o = (part ? out1 : out0) + s * out_stride + (size_t)j * N;
      const uint32_t* aA = part ? adA1 : adA0;
      const uint32_t* aB = part ? adB1 : adB0;
      const uint32_t* a = aA ? aA + b * adA_stride + (size_t)j * N : nullptr;
      const uint32_t* c = aB ? aB + s * adB_stride + (size_t)j * N : nullptr;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int idx = tid + e * NT;
        uint32_t v = md.subp(acc0[e]);
        if (a) v = md.subp(v + a[idx]);
        if (c) v = md.subp(v + c[idx]);
        o[idx] = v;
      }
    }
  }
}

template <int LOGN, int LE>
static int run_ks_plain(hefv_ctx* c, const uint32_t* kb, const uint32_t* km, const uint32_t* dig,
                        int64_t ds, uint32_t* o0, uint32_t* o1, int64_t os, const int32_t* slot,
                        const uint32_t* a0, const uint32_t* a1, int64_t as, const uint32_t* b0,
                        const uint32_t* b1, int64_t bs, int64_t B, cudaStream_t st);

template <int LOGN>
static int run_ks(hefv_ctx* c, const uint32_t* kb, const uint32_t* km, const uint32_t* dig,
                  int64_t ds, uint32_t* o0, uint32_t* o1, int64_t os, const int32_t* slot,
                  const uint32_t* a0, const uint32_t* a1, int64_t as, const uint32_t* b0,
                  const uint32_t* b1, int64_t bs, int64_t B, cudaStream_t st) {
  return run_ks_plain<LOGN, KsLoge<LOGN>::v>(c, kb, km, dig, ds, o0, o1, os, slot, a0, a1, as, b0,
                                             b1, bs, B, st);
}

template <int LOGN, int LE>
static int run_ks_plain(hefv_ctx* c, const uint32_t* kb, const uint32_t* km, const uint32_t* dig,
                        int64_t ds, uint32_t* o0, uint32_t* o1, int64_t os, const int32_t* slot,
                        const uint32_t* a0, const uint32_t* a1, int64_t as, const uint32_t* b0,
                        const uint32_t* b1, int64_t bs, int64_t B, cudaStream_t st) {
  typedef Geo<LOGN, LE> G_;
  auto kern = k_keyswitch<LOGN, LE>;
  const size_t smem = (size_t)(1 << (LOGN - G_::RLAST)) * sizeof(uint2) +
                      ((size_t)G_::N + (size_t)((spad_size(G_::N) + 3) & ~3)) * 4 + 16;
  if (smem > 48 * 1024) {
    HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  const int64_t chunk = 65535ll * KS_CTS_PER_CTA;
  for (int64_t b0i = 0; b0i < B; b0i += chunk) {
    const int64_t nb = (B - b0i) < chunk ? (B - b0i) : chunk;
    dim3 grid(c->k, (unsigned)((nb + KS_CTS_PER_CTA - 1) / KS_CTS_PER_CTA));
    kern<<<grid, G_::NT, smem, st>>>(kb, km, dig + b0i * ds, ds, o0, o1, os,
                                     slot ? slot + b0i : nullptr, a0 ? a0 + b0i * as : nullptr,
                                     a1 ? a1 + b0i * as : nullptr, as, b0, b1, bs, nb, c->k,
                                     c->d_tw32, c->d_itw32, c->d_info32);
    HEFV_LAUNCH_CHECK("k_keyswitch");
    if (!slot && nb < B) {
      // without a slot map the output index equals the batch index: shift bases
      o0 += nb * os;
      o1 += nb * os;
      if (b0) b0 += nb * bs;
      if (b1) b1 += nb * bs;
    }
  }
  return 0;
}

}  // namespace hefv

using namespace hefv;

extern "C" int hefv_keyswitch(hefv_ctx* c, const uint32_t* kbody, const uint32_t* kmask,
                              const uint32_t* digits, int64_t dig_stride, uint32_t* out0,
                              uint32_t* out1, int64_t out_stride, const int32_t* slot,
                              const uint32_t* adA0, const uint32_t* adA1, int64_t adA_stride,
                              const uint32_t* adB0, const uint32_t* adB1, int64_t adB_stride,
                              int64_t B, void* stream) {
  if (!c || !c->fv_ready) return fail("hefv_keyswitch: context without FV setup");
  if (B <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  ks_begin(c, B, st);
  int r;
  switch (c->log_n) {
#define HEFV_KS(L)                                                                              \
  case L:                                                                                       \
    r = run_ks<L>(c, kbody, kmask, digits, dig_stride, out0, out1, out_stride, slot, adA0,    \
                  adA1, adA_stride, adB0, adB1, adB_stride, B, st);                             \
    break;
    HEFV_KS(4)
    HEFV_KS(5)
    HEFV_KS(6)
    HEFV_KS(7)
    HEFV_KS(8)
    HEFV_KS(9)
    HEFV_KS(10)
    HEFV_KS(11)
    HEFV_KS(12)
    HEFV_KS(13)
    HEFV_KS(14)
#undef HEFV_KS
    default:
      r = fail("hefv_keyswitch: unsupported N");
  }
  ks_end(c, st);
  return r;
}
