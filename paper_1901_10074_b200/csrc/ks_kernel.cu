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

template <int LOGN>
struct KsLoge {
  static constexpr int v = LOGN >= 14 ? 5 : 4;
};

template <int LOGN, int LOGE>
__global__ void __launch_bounds__(Geo<LOGN, LOGE>::NT)
    k_keyswitch(const uint32_t* __restrict__ kbody, const uint32_t* __restrict__ kmask,
                const uint32_t* __restrict__ digits, int64_t dig_stride, uint32_t* out0,
                uint32_t* out1, int64_t out_stride, const int32_t* __restrict__ slot,
                const uint32_t* __restrict__ adA0, const uint32_t* __restrict__ adA1,
                int64_t adA_stride, const uint32_t* adB0, const uint32_t* adB1, int64_t adB_stride,
                int k, const uint2* __restrict__ tw_all, const uint2* __restrict__ itw_all,
                const Prime32Info* __restrict__ info) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int E = G_::E;
  constexpr int NT = G_::NT;
  constexpr int N = G_::N;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smraw);
  const int j = blockIdx.x;
  const int64_t b = blockIdx.y;
  const int tid = threadIdx.x;
  const Prime32Info inf = info[j];
  const Mod32 md = make_mod(inf);
  const uint2* tw = tw_all + (size_t)j * N;
  const uint32_t* dig = digits + b * dig_stride;

  uint32_t acc0[E], acc1[E], x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc0[e] = acc1[e] = 0u;

  for (int i = 0; i < k; ++i) {
    const uint32_t* src = dig + (size_t)i * N;
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = __ldg(src + tid + e * NT);
    cta_fwd<LOGN, LOGE, Mod32>(md, x, sm, tw);
    const size_t koff = ((size_t)j * k + i) * N + (size_t)tid * E;
    const uint4* kb = reinterpret_cast<const uint4*>(kbody + koff);
    const uint4* km = reinterpret_cast<const uint4*>(kmask + koff);
#pragma unroll
    for (int v = 0; v < E / 4; ++v) {
      const uint4 wb = __ldg(kb + v);
      const uint4 wm = __ldg(km + v);
      const uint32_t bb[4] = {wb.x, wb.y, wb.z, wb.w};
      const uint32_t mm[4] = {wm.x, wm.y, wm.z, wm.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = v * 4 + q;
        acc0[e] = md.sub2p(acc0[e] + mont_mul_lazy(x[e], bb[q], inf.p, inf.pinv_neg));
        acc1[e] = md.sub2p(acc1[e] + mont_mul_lazy(x[e], mm[q], inf.p, inf.pinv_neg));
      }
    }
  }

  const int64_t s = slot ? (int64_t)slot[b] : b;
  const uint2* itw = itw_all + (size_t)j * N;
  // part 0
  cta_inv<LOGN, LOGE, Mod32>(md, acc0, sm, itw, inf.ninv, inf.wn);
  {
    uint32_t* o = out0 + s * out_stride + (size_t)j * N;
    const uint32_t* a = adA0 ? adA0 + b * adA_stride + (size_t)j * N : nullptr;
    const uint32_t* c = adB0 ? adB0 + s * adB_stride + (size_t)j * N : nullptr;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int idx = tid + e * NT;
      uint32_t v = md.subp(acc0[e]);
      if (a) v = md.subp(v + a[idx]);
      if (c) v = md.subp(v + c[idx]);
      o[idx] = v;
    }
  }
  __syncthreads();
  cta_inv<LOGN, LOGE, Mod32>(md, acc1, sm, itw, inf.ninv, inf.wn);
  {
    uint32_t* o = out1 + s * out_stride + (size_t)j * N;
    const uint32_t* a = adA1 ? adA1 + b * adA_stride + (size_t)j * N : nullptr;
    const uint32_t* c = adB1 ? adB1 + s * adB_stride + (size_t)j * N : nullptr;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int idx = tid + e * NT;
      uint32_t v = md.subp(acc1[e]);
      if (a) v = md.subp(v + a[idx]);
      if (c) v = md.subp(v + c[idx]);
      o[idx] = v;
    }
  }
}

template <int LOGN>
static int run_ks(hefv_ctx* c, const uint32_t* kb, const uint32_t* km, const uint32_t* dig,
                  int64_t ds, uint32_t* o0, uint32_t* o1, int64_t os, const int32_t* slot,
                  const uint32_t* a0, const uint32_t* a1, int64_t as, const uint32_t* b0,
                  const uint32_t* b1, int64_t bs, int64_t B, cudaStream_t st) {
  constexpr int LE = KsLoge<LOGN>::v;
  typedef Geo<LOGN, LE> G_;
  auto kern = k_keyswitch<LOGN, LE>;
  const size_t smem = (size_t)spad_size(G_::N) * 4;
  if (smem > 48 * 1024) {
    HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  for (int64_t b0i = 0; b0i < B; b0i += 65535) {
    const int64_t nb = (B - b0i) < 65535 ? (B - b0i) : 65535;
    dim3 grid(c->k, (unsigned)nb);
    kern<<<grid, G_::NT, smem, st>>>(kb, km, dig + b0i * ds, ds, o0, o1, os,
                                     slot ? slot + b0i : nullptr, a0 ? a0 + b0i * as : nullptr,
                                     a1 ? a1 + b0i * as : nullptr, as, b0, b1, bs, c->k,
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
  switch (c->log_n) {
#define HEFV_KS(L)                                                                              \
  case L:                                                                                       \
    return run_ks<L>(c, kbody, kmask, digits, dig_stride, out0, out1, out_stride, slot, adA0, \
                     adA1, adA_stride, adB0, adB1, adB_stride, B, st);
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
      return fail("hefv_keyswitch: unsupported N");
  }
}
