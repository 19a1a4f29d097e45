// Standalone batched negacyclic NTTs (K1/K2 for 30-bit primes, K3 for
// 64-bit primes): each polynomial resident in one CTA's registers + one
// padded shared tile (ntt.cuh).  Replaces NttPrime.fwd/inv (reference
// ntt.py:191-224) including the object-dtype path for p >= 2^31.
//   * k_ntt32_b / k_ntt64_b: persistent prime-major CTAs (device order);
//   * k_ntt_fwd / k_ntt_inv: one CTA per polynomial (natural order, small N,
//     and the 64-bit sizes where that measured faster);
//   * k_ntt64_top + k_ntt64_sub: 64-bit N = 2^15 / 2^16 (and the 2^14
//     forward) as an outer-stage streaming pass plus 2^12-point sub-transforms;
//   * k_ntt32_top + k_ntt32_b<14, ., SUB>: 30-bit N = 2^16 the same way;
//   * k_ntt_cl_fwd: 30-bit N = 2^15 rows of the 64-bit key switch's aux basis as
//     one 2-CTA thread-block cluster each, the CTA-spanning exchange through
//     distributed shared memory;
#include <cstdlib>

#include "../../include/hefv.h"
#include "internal.h"
#include "ntt.cuh"
#include "kcommon.cuh"
#include "cluster.cuh"

namespace hefv {

#ifndef NTT64_ROWIO
#define NTT64_ROWIO 1  // 64-bit row-layout global I/O through warp-contiguous chunks
#endif

// transform input -> lazy range: 64-bit primes any u64; 30-bit primes from
// u32 or from u64 < 2^62 (the 64-bit key switch's digits)
__device__ __forceinline__ uint64_t cl_in(uint64_t v, const Prime64Info& i) {
  return v >= i.p ? barrett64(v, i.p, i.mu) : v;
}
__device__ __forceinline__ uint32_t cl_in(uint64_t v, const Prime32Info& i) {
  return barrett62(v, i.p, i.mu);
}
__device__ __forceinline__ uint32_t cl_in(uint32_t v, const Prime32Info& i) {
  return barrett62(v, i.p, i.mu);
}

template <int LOGN, int LOGE, class M, class TIn = typename M::T>
__global__ void __launch_bounds__(Geo<LOGN, LOGE>::NT)
    k_ntt_fwd(const TIn* __restrict__ in, typename M::T* __restrict__ out, int nprimes,
              int prime_base, int natural, const typename M::Tw* __restrict__ tw_all,
              const typename InfoOf<M>::I* __restrict__ info, int bcast) {
  typedef Geo<LOGN, LOGE> G_;
  typedef typename M::T T;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const size_t poly = blockIdx.x;
  const int pi = prime_base + (int)(poly % nprimes);
  const auto inf = info[pi];
  const M md = make_mod(inf);
  const typename M::Tw* tw = tw_all + (size_t)pi * G_::N;
  // bcast: one input row per batch index, transformed under every prime
  const TIn* src = in + (bcast ? poly / nprimes : poly) * G_::N;
  T* dst = out + poly * G_::N;
  const int tid = threadIdx.x;
  T x[G_::E];
#pragma unroll
  for (int e = 0; e < G_::E; ++e) x[e] = cl_in(src[tid + e * G_::NT], inf);
  cta_fwd<LOGN, LOGE, M>(md, x, sm, tw);
#pragma unroll
  for (int e = 0; e < G_::E; ++e) x[e] = md.canon4(x[e]);
  if (!natural) {
    if constexpr (sizeof(T) == 8 && LOGE == 4 && G_::NT >= 32 && NTT64_ROWIO) {
      uint4 c[8];  // warp-contiguous 128-bit stores (see k_ntt64_sub)
      warp_rows_to_chunks64(warp_tile_region(sm, tid), tid & 31, x, c);
      uint4* d4 = reinterpret_cast<uint4*>(dst + (tid >> 5) * 512) + (tid & 31);
#pragma unroll
      for (int i = 0; i < 8; ++i) d4[32 * i] = c[i];
    } else {
      store_row_vec<LOGN, LOGE, T>(dst, tid, x);
    }
  } else {
    // dev index i holds natural index bitrev(i): stage through smem
    __syncthreads();
#pragma unroll
    for (int e = 0; e < G_::E; ++e) sm[spad(brev_n(row_index<LOGN, LOGE>(tid, e), LOGN))] = x[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < G_::E; ++e) dst[tid + e * G_::NT] = sm[spad(tid + e * G_::NT)];
  }
}

template <int LOGN, int LOGE, class M>
__global__ void __launch_bounds__(Geo<LOGN, LOGE>::NT)
    k_ntt_inv(const typename M::T* __restrict__ in, typename M::T* __restrict__ out, int nprimes,
              int prime_base, int natural, const typename M::Tw* __restrict__ itw_all,
              const typename InfoOf<M>::I* __restrict__ info) {
  typedef Geo<LOGN, LOGE> G_;
  typedef typename M::T T;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const size_t poly = blockIdx.x;
  const int pi = prime_base + (int)(poly % nprimes);
  const auto inf = info[pi];
  const M md = make_mod(inf);
  const typename M::Tw* itw = itw_all + (size_t)pi * G_::N;
  const T* src = in + poly * G_::N;
  T* dst = out + poly * G_::N;
  const int tid = threadIdx.x;
  T x[G_::E];
  if (!natural) {
    if constexpr (sizeof(T) == 8 && LOGE == 4 && G_::NT >= 32 && NTT64_ROWIO) {
      uint4 c[8];  // warp-contiguous 128-bit loads (see k_ntt64_sub); the tile is unused yet
      const uint4* s4 = reinterpret_cast<const uint4*>(src + (tid >> 5) * 512) + (tid & 31);
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = __ldg(s4 + 32 * i);
      warp_chunks_to_rows64(warp_tile_region(sm, tid), tid & 31, c, x);
    } else {
      load_row_vec<LOGN, LOGE, T>(src, tid, x);
    }
  } else {
#pragma unroll
    for (int e = 0; e < G_::E; ++e)
      sm[spad(brev_n(tid + e * G_::NT, LOGN))] = src[tid + e * G_::NT];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < G_::E; ++e) x[e] = sm[spad(row_index<LOGN, LOGE>(tid, e))];
    __syncthreads();
  }
  cta_inv<LOGN, LOGE, M>(md, x, sm, itw, inf.ninv, inf.wn);
#pragma unroll
  for (int e = 0; e < G_::E; ++e) dst[tid + e * G_::NT] = md.subp(x[e]);
}

// ---- batched device-order path for 32-bit primes, N >= 2^10 ---------------
// Persistent: one wave of CTAs (as many per SM as fit), CTA c owns the range
// [c P / G, (c+1) P / G) of the P = batch x nprimes polynomials in prime-major
// order, so every SM gets the same number of transforms (no partial last
// wave) and restages twiddles only at a prime boundary.  The prime's Shoup
// twiddles of the full passes live in shared memory; each polynomial is
// bulk-copied (cp.async.bulk) into a staging buffer one transform ahead (the
// copy is issued right after the current transform's first CTA barrier).

// LASTSM (forward): the last pass's twiddles (entries [NTW, N), 48 KB at
// 2^14) also live in shared memory, as single-word Montgomery forms (the
// Shoup pairs would not fit next to the tile and the stage); the last pass
// then uses Montgomery products instead of L2-latency-bound Shoup loads.
// N with the last pass's twiddles in shared memory (2^12: inverse 0.60 ->
// 0.63 of the butterfly peak, forward unchanged; measured on a B200)
#ifndef NTT32_LASTSM_MASK
#define NTT32_LASTSM_MASK ((1 << 14) | (1 << 12))
#endif
#ifndef NTT32_ALLSM_MASK
// N whose whole Shoup table (8 N bytes) is staged in shared memory: at 2^12 a third
// of the butterflies are in the last pass, and Shoup pairs for it (3 CTAs of 65 KB
// per SM) beat the Montgomery words (4 CTAs of 50 KB): forward 0.588 -> 0.604
#define NTT32_ALLSM_MASK (1 << 12)
#endif
#ifndef ROWSTORE_T
#define ROWSTORE_T 1  // forward output through warp_rows_to_chunks (coalesced 128-bit stores)
#endif
#ifndef NTT32_MINB_SMALL
#define NTT32_MINB_SMALL 0  // 0: 1024 / NT resident CTAs per SM for N <= 2^12
#endif
template <int LOGN>
constexpr int ntt32_minb() {
  if (((NTT32_ALLSM_MASK >> LOGN) & 1) && LOGN == 12) return 3;  // 65 KB per CTA
  return (Geo<LOGN, 4>::NT <= 256 && NTT32_MINB_SMALL) ? NTT32_MINB_SMALL
                                                       : 1024 / Geo<LOGN, 4>::NT;
}

template <int LOGN, bool FWD>
struct Ntt32B {
  typedef Geo<LOGN, 4> G_;
  // fwd: last pass; inv: its first pass
  static constexpr bool ALLSM = ((NTT32_ALLSM_MASK >> LOGN) & 1) != 0;
  static constexpr bool LASTSM = !ALLSM && ((NTT32_LASTSM_MASK >> LOGN) & 1) != 0;
  static constexpr int NTW = ALLSM ? G_::N : 1 << (LOGN - G_::RLAST);
  static constexpr size_t smem = (size_t)NTW * sizeof(uint2) +
                                 (size_t)((spad_size(G_::N) + 3) & ~3) * 4 + (size_t)G_::N * 4 +
                                 16 + (LASTSM ? (size_t)(G_::N - NTW) * 4 : 0);
};

// SUB (N = 2^14 only): the polynomials are the 2^log_s sub-blocks of 2^(14 + log_s)-
// point ones (k_ntt32_top ran, or will run, the log_s outer stages): work items
// walk (prime, sub-block, batch), the staged tables are the sub-block's slices of
// the large transform's tables (entry idx of the virtual table is entry
// idx + ((2^log_s + g - 1) << floor(log2 idx)) of the real one), forward inputs
// arrive lazily reduced (< 4p) and inverse outputs leave lazily reduced (< 2p,
// N^-1 is merged by the outer pass).
template <int LOGN, bool FWD, bool SUB = false>
__global__ void __launch_bounds__(Geo<LOGN, 4>::NT, ntt32_minb<LOGN>())
    k_ntt32_b(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int64_t batch,
              int nprimes, int prime_base, const uint2* __restrict__ tw_all,
              const Prime32Info* __restrict__ info, const uint32_t* __restrict__ twm_all,
              int log_s = 0) {
  typedef Geo<LOGN, 4> G_;
  constexpr int E = G_::E;
  constexpr int NT = G_::NT;
  constexpr int N = G_::N;
  constexpr int NTW = Ntt32B<LOGN, FWD>::NTW;
  constexpr bool LASTSM = Ntt32B<LOGN, FWD>::LASTSM;
  constexpr bool ALLSM = Ntt32B<LOGN, FWD>::ALLSM;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint2* tws = reinterpret_cast<uint2*>(smraw);
  uint32_t* sm = reinterpret_cast<uint32_t*>(tws + NTW);
  uint32_t* stage = sm + ((spad_size(N) + 3) & ~3);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stage + N);
  uint32_t* twl = reinterpret_cast<uint32_t*>(mbar + 2);  // LASTSM: entries [NTW, N)
  const int tid = threadIdx.x;
  const int nsub = SUB ? 1 << log_s : 1;
  const int64_t P = batch * nprimes * nsub;
  const int64_t qbeg = P * blockIdx.x / gridDim.x;
  const int64_t qend = P * (blockIdx.x + 1) / gridDim.x;
  if (qbeg >= qend) return;
  // prime-major work order q -> (prime j, [sub-block g,] batch index b); memory is
  // (b, j, N) (SUB: (b, j, g, N))
  auto poly = [&](int64_t q) {
    const int64_t jg = q / batch, b = q - jg * batch;
    if constexpr (SUB) {
      const int64_t j = jg >> log_s, g = jg - (j << log_s);
      return ((b * nprimes + j) * nsub + g) * (int64_t)N;
    } else {
      return (b * nprimes + jg) * (int64_t)N;
    }
  };
  if (tid == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) bulk_g2s(stage, in + poly(qbeg), N * 4, mbar);
  uint32_t phase = 0;
  int cur = -1;
  Prime32Info inf;
  const uint2* twg = nullptr;
  for (int64_t q = qbeg; q < qend; ++q) {
    const int jg = (int)(q / batch);  // prime (SUB: prime * nsub + sub-block)
    if (jg != cur) {  // (re)stage this prime's (sub-block's) twiddles
      cur = jg;
      const int j = SUB ? jg >> log_s : jg;
      inf = info[prime_base + j];
      twg = tw_all + (size_t)(prime_base + j) * (SUB ? (size_t)N << log_s : (size_t)N);
      __syncthreads();  // the previous table is no longer read
      if constexpr (SUB) {
        static_assert(!SUB || LASTSM, "the sub-block form stages both table parts");
        const uint32_t bm1 = (uint32_t)(nsub + (jg - (j << log_s)) - 1);  // base - 1
        const uint32_t* twmg = twm_all + (size_t)(prime_base + j) * ((size_t)N << log_s);
        for (int i = tid; i < NTW; i += NT)
          tws[i] = __ldg(twg + (i ? i + (bm1 << (31 - __clz(i))) : 0));
        for (int i = NTW + tid; i < N; i += NT)
          twl[i - NTW] = __ldg(twmg + i + (bm1 << (31 - __clz(i))));
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(twg);
        uint4* dst = reinterpret_cast<uint4*>(tws);
        for (int i = tid; i < NTW / 2; i += NT) dst[i] = __ldg(src + i);
        if constexpr (LASTSM) {
          const uint4* srcm =
              reinterpret_cast<const uint4*>(twm_all + (size_t)(prime_base + j) * N + NTW);
          uint4* dstm = reinterpret_cast<uint4*>(twl);
          for (int i = tid; i < (N - NTW) / 4; i += NT) dstm[i] = __ldg(srcm + i);
        }
      }
      __syncthreads();
    }
    const Mod32 md{inf.p, 2 * inf.p};
#if !(HEFV_DIAG & 16)
    mbar_wait(mbar, phase);
    phase ^= 1u;
#endif
    uint32_t x[E];
#if HEFV_DIAG & 16
    const uint32_t* nxt = nullptr;
#else
    const uint32_t* nxt = q + 1 < qend ? in + poly(q + 1) : nullptr;
#endif
    auto hook = [&]() {
      if (tid == 0 && nxt) bulk_g2s(stage, nxt, N * 4, mbar);
    };
    if constexpr (FWD) {
      // input -> [0, 4p): the prime's class is uniform, so branch once around
      // the 16 loads (a per-element branch costs ~8 issue slots per word)
      if (HEFV_DIAG & 16) {
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = (uint32_t)(tid * 977 + e * 131 + (int)q);
      } else if (SUB || inf.p >= (1u << 30)) {
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = stage[tid + e * NT];
      } else if (inf.p > (1u << 29)) {
        const uint32_t p4 = 4 * inf.p;  // x < 2^32 < 8p: one conditional subtraction
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t v = stage[tid + e * NT];
          x[e] = min(v, v - p4);
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = barrett62(stage[tid + e * NT], inf.p, inf.mu);
      }
      if constexpr (LASTSM && LOGN == 14) {
        // butterfly sums on the ALU pipe (Mod32A / Mod32MA, modarith.cuh)
        const Mod32A ma(inf.p);
        cta_fwd<LOGN, 4, Mod32A, decltype(hook), false>(ma, x, sm, tws, twg, hook);
        const Mod32MA mm(inf.p, inf.pinv, ma.ones);
        fwd_last_pass<LOGN, 4, Mod32MA>(mm, x, tid, twl - NTW);
      } else if constexpr (LASTSM) {
        cta_fwd<LOGN, 4, Mod32, decltype(hook), false>(md, x, sm, tws, twg, hook);
        const Mod32M mm{inf.p, 2 * inf.p, inf.pinv};
        fwd_last_pass<LOGN, 4, Mod32M>(mm, x, tid, twl - NTW);
      } else if constexpr (ALLSM) {
        cta_fwd<LOGN, 4, Mod32>(md, x, sm, tws, nullptr, hook);
      } else {
        cta_fwd<LOGN, 4, Mod32>(md, x, sm, tws, twg, hook, LOGN - G_::RLAST);
      }
#if HEFV_DIAG & 8
      uint32_t acc = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) acc ^= x[e];
      if (acc == 0x12345u) out[poly(q) + tid] = acc;
#else
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = md.canon4(x[e]);
      if constexpr (NT >= 32 && ROWSTORE_T) {
        uint4 c[4];
        warp_rows_to_chunks(warp_tile_region(sm, tid), tid & 31, x, c);
        uint4* dst = reinterpret_cast<uint4*>(out + poly(q) + (tid >> 5) * 512) + (tid & 31);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[32 * i] = c[i];
      } else {
        store_row_vec<LOGN, 4, uint32_t>(out + poly(q), tid, x);
      }
#endif
    } else {
#if HEFV_DIAG & 16
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = (uint32_t)(tid * 977 + e * 131 + (int)q) & 0xfffffffu;
#else
      load_row16_smem(stage, tid, x);
#endif
      if constexpr (LASTSM) {
        const Mod32M mm{inf.p, 2 * inf.p, inf.pinv};
        inv_last_pass<LOGN, 4, Mod32M>(mm, x, tid, twl - NTW, 0u, 0u);  // N^-1 is in pass 0
        cta_inv<LOGN, 4, Mod32, decltype(hook), false, SUB>(md, x, sm, tws, inf.ninv, inf.wn, twg,
                                                            hook);
      } else if constexpr (ALLSM) {
        cta_inv<LOGN, 4, Mod32>(md, x, sm, tws, inf.ninv, inf.wn, nullptr, hook);
      } else {
        cta_inv<LOGN, 4, Mod32>(md, x, sm, tws, inf.ninv, inf.wn, twg, hook);
      }
      uint32_t* dst = out + poly(q);
#if HEFV_DIAG & 8
      uint32_t acc = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) acc ^= x[e];
      if (acc == 0x12345u) dst[tid] = acc;
#else
#pragma unroll
      for (int e = 0; e < E; ++e) dst[tid + e * NT] = SUB ? x[e] : md.subp(x[e]);
#endif
    }
  }
}

// ---- batched device-order path for 64-bit primes, 2^10 <= N <= 2^14 --------
// Same persistent prime-major schedule as k_ntt32_b.  STAGE: the prime's
// full-pass twiddles (16-byte Shoup pairs) are staged in shared memory next
// to the tile (64 KB at N = 2^14; loading them from L2 inside the passes
// left the 2^14 transform long-scoreboard bound).  The next polynomial is
// prefetched into L2 by one bulk prefetch per transform; a shared staging
// copy as in k_ntt32_b does not fit next to a 64-bit tile.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int LOGN>
struct Ntt64B {
  typedef Geo<LOGN, 4> G_;
  static constexpr int NTW = 1 << (LOGN - G_::RLAST);
  static constexpr size_t tw_bytes(bool stage) { return stage ? (size_t)NTW * 16 : 0; }
  static constexpr size_t smem(bool stage) {
    return tw_bytes(stage) + (size_t)((spad_size(G_::N) + 1) & ~1) * 8;
  }
};

template <int LOGN, bool FWD, bool STAGE>
__global__ void __launch_bounds__(Geo<LOGN, 4>::NT, LOGN >= 13 ? 1024 / Geo<LOGN, 4>::NT : 2)
    k_ntt64_b(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int64_t batch,
              int nprimes, int prime_base, const ulonglong2* __restrict__ tw_all,
              const Prime64Info* __restrict__ info, int bcast) {
  typedef Geo<LOGN, 4> G_;
  constexpr int E = G_::E;
  constexpr int NT = G_::NT;
  constexpr int N = G_::N;
  constexpr int NTW = Ntt64B<LOGN>::NTW;
  extern __shared__ __align__(16) unsigned char smraw[];
  ulonglong2* tws = reinterpret_cast<ulonglong2*>(smraw);
  uint64_t* sm = reinterpret_cast<uint64_t*>(smraw + Ntt64B<LOGN>::tw_bytes(STAGE));
  const int tid = threadIdx.x;
  const int64_t P = batch * nprimes;
  const int64_t qbeg = P * blockIdx.x / gridDim.x;
  const int64_t qend = P * (blockIdx.x + 1) / gridDim.x;
  if (qbeg >= qend) return;
  // prime-major work order q -> (prime j, batch index b), walked without
  // divisions (a 64-bit division is a call that forces spills here)
  int j = (int)(qbeg / batch);
  int64_t b = qbeg - (int64_t)j * batch;
  const int64_t pstride = (int64_t)nprimes * N;
  const Prime64Info* ip = nullptr;
  const ulonglong2* twg = nullptr;
  uint64_t p = 0;
  for (int64_t q = qbeg; q < qend; ++q) {
    if (ip == nullptr || b == batch) {
      if (ip != nullptr) {
        b = 0;
        ++j;
      }
      ip = info + prime_base + j;
      p = ip->p;
      twg = tw_all + (size_t)(prime_base + j) * N;
      if constexpr (STAGE) {
        __syncthreads();  // the previous prime's table is no longer read
        for (int i = tid; i < NTW; i += NT) tws[i] = __ldg(twg + i);
        __syncthreads();
      }
    }
    const uint64_t* src = bcast ? in + b * N : in + b * pstride + (int64_t)j * N;
    uint64_t* dst = out + b * pstride + (int64_t)j * N;
    if (tid == 0 && q + 1 < qend) {
      const bool wrap = b + 1 == batch;
      bulk_prefetch_l2(bcast ? (wrap ? in : src + N)
                             : (wrap ? in + (j + 1) * (int64_t)N : src + pstride), N * 8);
    }
    ++b;
    const Mod64 md{p, 2 * p};
    const ulonglong2* twf = STAGE ? tws : twg;
    uint64_t x[E];
    if constexpr (FWD) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint64_t v = src[tid + e * NT];
        x[e] = v >= p ? barrett64(v, p, ip->mu) : v;
      }
      cta_fwd<LOGN, 4, Mod64>(md, x, sm, twf, twg, NoHook(), LOGN - G_::RLAST);
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = md.canon4(x[e]);
      if constexpr (NTT64_ROWIO) {
        uint4 c[8];  // warp-contiguous 128-bit stores (see k_ntt64_sub)
        warp_rows_to_chunks64(warp_tile_region(sm, tid), tid & 31, x, c);
        uint4* d4 = reinterpret_cast<uint4*>(dst + (tid >> 5) * 512) + (tid & 31);
#pragma unroll
        for (int i = 0; i < 8; ++i) d4[32 * i] = c[i];
      } else {
        store_row_vec<LOGN, 4, uint64_t>(dst, tid, x);
      }
    } else {
      // (2^13: the chunk registers spill at 64 registers per thread, 0.659 -> 0.626, and one
      // 512-thread CTA per SM at 128 registers loses more: 0.745 / 0.660 -> 0.717 / 0.649)
      if constexpr (NTT64_ROWIO && LOGN == 14) {
        uint4 c[8];
        const uint4* s4 = reinterpret_cast<const uint4*>(src + (tid >> 5) * 512) + (tid & 31);
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = __ldg(s4 + 32 * i);
        __syncthreads();  // the previous transform's last exchange has been read
        warp_chunks_to_rows64(warp_tile_region(sm, tid), tid & 31, c, x);
      } else {
        load_row_vec<LOGN, 4, uint64_t>(src, tid, x);
      }
      cta_inv<LOGN, 4, Mod64>(md, x, sm, twf, ip->ninv, ip->wn, twg);
#pragma unroll
      for (int e = 0; e < E; ++e) dst[tid + e * NT] = md.subp(x[e]);
    }
  }
}

static int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
  }
  return n;
}

// ---- 64-bit transforms of 2^13 .. 2^16 points as two HBM passes -------------
// A 64-bit transform holds its 16 words per thread in 32 registers, so the
// one-CTA (1024 threads, 64 registers) and cluster forms above 2^12 run
// register-starved (0.52-0.67 of the butterfly peak) while the 2^12 transform
// (256 threads, up to 128 registers, several CTAs per SM) reaches 0.82.  The
// split form runs the S = LOGN - 12 outermost stages as a streaming pass over
// HBM (k_ntt64_top: 2^S words per thread at stride N / 2^S, coalesced, the
// 2^S - 1 twiddles uniform) and the remaining 12 stages as 2^S independent
// 2^12-point sub-transforms per polynomial (k_ntt64_sub: the CTA-resident
// transform with table entries (2^S + g) << stage for sub-block g).  Same
// butterfly network and table as the one-kernel forms, hence the same device
// order and the same canonical outputs.
template <int S, bool FWD>
__global__ void __launch_bounds__(256)
    k_ntt64_top(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int nprimes,
                int prime_base, int log_n, const ulonglong2* __restrict__ tw_all,
                const Prime64Info* __restrict__ info, int bcast) {
  constexpr int R = 1 << S;
  const int64_t n = (int64_t)1 << log_n;
  const int64_t ns = n >> S;                 // element stride between a thread's words
  const int chunks = (int)(ns >> 8);         // 256-thread blocks per polynomial
  const int64_t q = blockIdx.x / chunks;     // polynomial (b, j), j fastest
  const int64_t idx = (int64_t)(blockIdx.x - q * chunks) * 256 + threadIdx.x;
  const int j = (int)(q % nprimes);
  const Prime64Info* ip = info + prime_base + j;
  const uint64_t p = ip->p;
  const Mod64 md{p, 2 * p};
  const ulonglong2* tw = tw_all + (size_t)(prime_base + j) * n;
  const uint64_t* src = in + (bcast ? q / nprimes : q) * n + idx;
  uint64_t* dst = out + q * n + idx;
  uint64_t x[R];
  if constexpr (FWD) {
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const uint64_t v = src[e * ns];
      x[e] = v >= p ? barrett64(v, p, ip->mu) : v;
    }
#pragma unroll
    for (int l = 0; l < S; ++l) {
      const int half = R >> (l + 1);
#pragma unroll
      for (int u = 0; u < (1 << l); ++u) {
        const ulonglong2 w = __ldg(tw + (1 << l) + u);
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) md.ct(x[u * 2 * half + e0], x[u * 2 * half + e0 + half], w);
      }
    }
#pragma unroll
    for (int e = 0; e < R; ++e) dst[e * ns] = x[e];  // lazy, < 4p
  } else {
#pragma unroll
    for (int e = 0; e < R; ++e) x[e] = src[e * ns];  // < 2p from k_ntt64_sub
#pragma unroll
    for (int l = S - 1; l >= 0; --l) {
      const int half = R >> (l + 1);
#pragma unroll
      for (int u = 0; u < (1 << l); ++u) {
        if (l == 0) {
#pragma unroll
          for (int e0 = 0; e0 < half; ++e0) md.gs_last(x[e0], x[e0 + half], ip->ninv, ip->wn);
        } else {
          const ulonglong2 w = __ldg(tw + (1 << l) + u);
#pragma unroll
          for (int e0 = 0; e0 < half; ++e0) md.gs(x[u * 2 * half + e0], x[u * 2 * half + e0 + half], w);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < R; ++e) dst[e * ns] = md.subp(x[e]);
  }
}

#ifndef NTT64_SUB_MINB
#define NTT64_SUB_MINB 2  // resident CTAs per SM the sub-transform is compiled for
#endif
// Persistent CTAs over the P = nprimes x 2^S x batch sub-blocks in (prime,
// sub-block, batch) order, so a CTA keeps one 64 KB twiddle slice hot in L1.
template <bool FWD>
__global__ void __launch_bounds__(256, NTT64_SUB_MINB)
    k_ntt64_sub(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int64_t batch,
                int nprimes, int prime_base, int log_s, const ulonglong2* __restrict__ tw_all,
                const Prime64Info* __restrict__ info) {
  typedef Geo<12, 4> G_;
  constexpr int E = G_::E;
  constexpr int NT = G_::NT;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(smraw);
  const int tid = threadIdx.x;
  const int nsub = 1 << log_s;
  const int64_t n = (int64_t)G_::N << log_s;
  const int64_t per_prime = (int64_t)nsub * batch;
  const int64_t P = per_prime * nprimes;
  const int64_t qbeg = P * blockIdx.x / gridDim.x;
  const int64_t qend = P * (blockIdx.x + 1) / gridDim.x;
  if (qbeg >= qend) return;
  int j = (int)(qbeg / per_prime);
  int64_t r = qbeg - (int64_t)j * per_prime;
  int g = (int)(r / batch);
  int64_t b = r - (int64_t)g * batch;
  const int64_t pstride = (int64_t)nprimes * n;
  for (int64_t q = qbeg; q < qend; ++q) {
    const Prime64Info* ip = info + prime_base + j;
    const uint64_t p = ip->p;
    const Mod64 md{p, 2 * p};
    const ulonglong2* tw = tw_all + (size_t)(prime_base + j) * n;
    const int64_t off = b * pstride + (int64_t)j * n + (int64_t)g * G_::N;
    const int base = nsub + g;
    // next work item (b fastest, then g, then j)
    if (++b == batch) {
      b = 0;
      if (++g == nsub) {
        g = 0;
        ++j;
      }
    }
    if (tid == 0 && q + 1 < qend)
      bulk_prefetch_l2(in + b * pstride + (int64_t)j * n + (int64_t)g * G_::N, G_::N * 8);
    uint64_t x[E];
    if constexpr (FWD) {
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = in[off + tid + e * NT];  // < 4p from k_ntt64_top
      cta_fwd<12, 4, Mod64>(md, x, sm, tw, nullptr, NoHook(), 0, base);
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = md.canon4(x[e]);
      // warp-contiguous 128-bit stores (a row-layout store puts each lane's 16
      // bytes in a different 128-byte line)
      uint4 c[8];
      warp_rows_to_chunks64(warp_tile_region(sm, tid), tid & 31, x, c);
      uint4* dst = reinterpret_cast<uint4*>(out + off + (tid >> 5) * 512) + (tid & 31);
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[32 * i] = c[i];
    } else {
      uint4 c[8];
      const uint4* src = reinterpret_cast<const uint4*>(in + off + (tid >> 5) * 512) + (tid & 31);
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = __ldg(src + 32 * i);
      __syncthreads();  // the previous transform's last exchange has been read
      warp_chunks_to_rows64(warp_tile_region(sm, tid), tid & 31, c, x);
      cta_inv<12, 4, Mod64, NoHook, true, true>(md, x, sm, tw, ip->ninv, ip->wn, nullptr, NoHook(),
                                                base);
#pragma unroll
      for (int e = 0; e < E; ++e) out[off + tid + e * NT] = x[e];  // lazy, < 2p
    }
  }
}

template <int S>
static int launch_split64_s(bool fwd, const uint64_t* in, uint64_t* out, int64_t batch, int nprimes,
                            int prime_base, const ulonglong2* tw, const Prime64Info* info,
                            cudaStream_t st, int bcast) {
  const int log_n = 12 + S;
  const int64_t polys = batch * nprimes;
  const int64_t top_blocks = polys * ((int64_t)1 << (log_n - S - 8));
  if (top_blocks > 0x7fffffff) return fail("ntt64: batch too large");
  const size_t smem = (size_t)((spad_size(4096) + 1) & ~1) * 8;
  auto sub = fwd ? k_ntt64_sub<true> : k_ntt64_sub<false>;
  HEFV_CUDA(cudaFuncSetAttribute(sub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sub, 256, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t P = polys << S;
  const int64_t slots = (int64_t)sm_count() * per_sm;
  const unsigned grid = (unsigned)(P < slots ? P : slots);
  if (fwd) {
    k_ntt64_top<S, true><<<(unsigned)top_blocks, 256, 0, st>>>(in, out, nprimes, prime_base, log_n,
                                                                tw, info, bcast);
    HEFV_LAUNCH_CHECK("k_ntt64_top");
    sub<<<grid, 256, smem, st>>>(out, out, batch, nprimes, prime_base, S, tw, info);
    HEFV_LAUNCH_CHECK("k_ntt64_sub");
  } else {
    if (bcast) return fail("ntt64: broadcast rows are a forward-only input form");
    sub<<<grid, 256, smem, st>>>(in, out, batch, nprimes, prime_base, S, tw, info);
    HEFV_LAUNCH_CHECK("k_ntt64_sub");
    k_ntt64_top<S, false><<<(unsigned)top_blocks, 256, 0, st>>>(out, out, nprimes, prime_base,
                                                                 log_n, tw, info, 0);
    HEFV_LAUNCH_CHECK("k_ntt64_top");
  }
  return 0;
}

static int launch_split64(int log_n, bool fwd, const uint64_t* in, uint64_t* out, int64_t batch,
                          int nprimes, int prime_base, const ulonglong2* tw,
                          const Prime64Info* info, cudaStream_t st, int bcast) {
  switch (log_n) {
    case 14: return launch_split64_s<2>(fwd, in, out, batch, nprimes, prime_base, tw, info, st, bcast);
    case 15: return launch_split64_s<3>(fwd, in, out, batch, nprimes, prime_base, tw, info, st, bcast);
    case 16: return launch_split64_s<4>(fwd, in, out, batch, nprimes, prime_base, tw, info, st, bcast);
    default: return fail("ntt64 split: N must be 2^14 .. 2^16");
  }
}

// Measured (B200, 60-bit, L = 8; fraction of the 64-bit butterfly peak, one-kernel
// form -> split): 2^16 fwd 0.546 -> 0.719, inv 0.516 -> 0.659; 2^15 0.607 -> 0.692,
// 0.608 -> 0.643; 2^14 fwd 0.641 -> 0.667 but inv 0.667 -> 0.630; 2^13 loses
// (0.656 -> 0.636, 0.659 -> 0.601): its single outer stage is not worth an HBM pass.
static bool ntt64_split(int log_n, bool fwd) { return log_n >= 15 || (log_n == 14 && fwd); }

template <int LOGN>
static int launch_b32(bool fwd, const uint32_t* in, uint32_t* out, int64_t batch, int nprimes,
                      int prime_base, const uint2* tw, const Prime32Info* info, cudaStream_t st,
                      const uint32_t* twm) {
  typedef Geo<LOGN, 4> G_;
  const size_t smem = fwd ? Ntt32B<LOGN, true>::smem : Ntt32B<LOGN, false>::smem;
  auto kern = fwd ? k_ntt32_b<LOGN, true> : k_ntt32_b<LOGN, false>;
  HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G_::NT, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t P = batch * nprimes;
  const int64_t slots = (int64_t)sm_count() * per_sm;
  const unsigned grid = (unsigned)(P < slots ? P : slots);
  kern<<<grid, G_::NT, smem, st>>>(in, out, batch, nprimes, prime_base, tw, info, twm, 0);
  HEFV_LAUNCH_CHECK("k_ntt32_b");
  return 0;
}

// 64-bit device-order transform variant: 0 = one CTA per polynomial
// (k_ntt_fwd/inv), 1 = persistent with twiddles from L1/L2.  The measured
// best per (N, direction) on a B200 (60-bit primes, L = 8, batch 256-1024):
// persistent for 2^13 and the 2^14 inverse (0.62-0.67 of the butterfly peak
// vs 0.57-0.61), one CTA per polynomial elsewhere.  (Staging the twiddles in
// shared memory never won and is not built.)
static int ntt64_mode(int log_n, bool fwd) {
  return (log_n == 13 || (log_n == 14 && !fwd)) ? 1 : 0;
}

template <int LOGN>
static int launch_b64(bool fwd, const uint64_t* in, uint64_t* out, int64_t batch, int nprimes,
                      int prime_base, const ulonglong2* tw, const Prime64Info* info, cudaStream_t st,
                      bool stage, int bcast) {
  typedef Geo<LOGN, 4> G_;
  const size_t smem = Ntt64B<LOGN>::smem(stage);
  auto kern = fwd ? k_ntt64_b<LOGN, true, false> : k_ntt64_b<LOGN, false, false>;
  HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G_::NT, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t P = batch * nprimes;
  const int64_t slots = (int64_t)sm_count() * per_sm;
  const unsigned grid = (unsigned)(P < slots ? P : slots);
  kern<<<grid, G_::NT, smem, st>>>(in, out, batch, nprimes, prime_base, tw, info, bcast);
  HEFV_LAUNCH_CHECK("k_ntt64_b");
  return 0;
}

// ---- 30-bit transforms of 2^15 / 2^16 points as two HBM passes ---------------
// The same split as the 64-bit one (k_ntt64_top / k_ntt64_sub): the S = LOGN - 14
// outermost stages stream over HBM, the remaining 14 run as 2^S sub-transforms
// in the persistent 2^14 kernel (k_ntt32_b<14, ., SUB>).  Replaces the
// 1024-thread x 32-word single CTA at 2^15 (0.37 / 0.43 of the butterfly peak)
// and the 4-CTA cluster at 2^16 (0.35 / 0.37) in device order.
template <int S, bool FWD, class TIn>
__global__ void __launch_bounds__(256)
    k_ntt32_top(const TIn* __restrict__ in, uint32_t* __restrict__ out, int nprimes,
                int prime_base, int log_n, const uint2* __restrict__ tw_all,
                const Prime32Info* __restrict__ info, int bcast) {
  constexpr int R = 1 << S;
  const int64_t n = (int64_t)1 << log_n;
  const int64_t ns = n >> S;
  const int chunks = (int)(ns >> 8);
  const int64_t q = blockIdx.x / chunks;  // polynomial (b, j), j fastest
  const int64_t idx = (int64_t)(blockIdx.x - q * chunks) * 256 + threadIdx.x;
  const int j = (int)(q % nprimes);
  const Prime32Info inf = info[prime_base + j];
  const Mod32 md{inf.p, 2 * inf.p};
  const uint2* tw = tw_all + (size_t)(prime_base + j) * n;
  uint32_t* dst = out + q * n + idx;
  uint32_t x[R];
  if constexpr (FWD) {
    const TIn* src = in + (bcast ? q / nprimes : q) * n + idx;
#pragma unroll
    for (int e = 0; e < R; ++e) x[e] = cl_in(src[e * ns], inf);
#pragma unroll
    for (int l = 0; l < S; ++l) {
      const int half = R >> (l + 1);
#pragma unroll
      for (int u = 0; u < (1 << l); ++u) {
        const uint2 w = __ldg(tw + (1 << l) + u);
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) md.ct(x[u * 2 * half + e0], x[u * 2 * half + e0 + half], w);
      }
    }
#pragma unroll
    for (int e = 0; e < R; ++e) dst[e * ns] = x[e];  // lazy, < 4p
  } else {
#pragma unroll
    for (int e = 0; e < R; ++e) x[e] = dst[e * ns];  // < 2p from the sub-transforms
#pragma unroll
    for (int l = S - 1; l >= 0; --l) {
      const int half = R >> (l + 1);
#pragma unroll
      for (int u = 0; u < (1 << l); ++u) {
        if (l == 0) {
#pragma unroll
          for (int e0 = 0; e0 < half; ++e0) md.gs_last(x[e0], x[e0 + half], inf.ninv, inf.wn);
        } else {
          const uint2 w = __ldg(tw + (1 << l) + u);
#pragma unroll
          for (int e0 = 0; e0 < half; ++e0) md.gs(x[u * 2 * half + e0], x[u * 2 * half + e0 + half], w);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < R; ++e) dst[e * ns] = md.subp(x[e]);
  }
}

// rows: polynomials per prime (bcast: input rows, each transformed under every prime)
template <int S, class TIn>
static int launch_split32(bool fwd, const TIn* in, uint32_t* out, int64_t rows, int nprimes,
                          int prime_base, const uint2* tw, const Prime32Info* info,
                          const uint32_t* twm, cudaStream_t st, int bcast) {
  const int log_n = 14 + S;
  const int64_t polys = rows * nprimes;
  if (polys <= 0) return 0;
  const int64_t top_blocks = polys << (log_n - S - 8);
  if (top_blocks > 0x7fffffff) return fail("ntt32: batch too large");
  const size_t smem = fwd ? Ntt32B<14, true>::smem : Ntt32B<14, false>::smem;
  auto sub = fwd ? k_ntt32_b<14, true, true> : k_ntt32_b<14, false, true>;
  HEFV_CUDA(cudaFuncSetAttribute(sub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t P = polys << S;
  const int64_t slots = sm_count();
  const unsigned grid = (unsigned)(P < slots ? P : slots);
  if (fwd) {
    k_ntt32_top<S, true, TIn><<<(unsigned)top_blocks, 256, 0, st>>>(in, out, nprimes, prime_base,
                                                                     log_n, tw, info, bcast);
    HEFV_LAUNCH_CHECK("k_ntt32_top");
    sub<<<grid, 1024, smem, st>>>(out, out, rows, nprimes, prime_base, tw, info, twm, S);
    HEFV_LAUNCH_CHECK("k_ntt32_b sub");
  } else {
    if constexpr (sizeof(TIn) != 4) {
      return fail("ntt32: wide rows are a forward-only input form");
    } else {
      if (bcast) return fail("ntt32: broadcast rows are a forward-only input form");
      sub<<<grid, 1024, smem, st>>>(in, out, rows, nprimes, prime_base, tw, info, twm, S);
      HEFV_LAUNCH_CHECK("k_ntt32_b sub");
      k_ntt32_top<S, false, uint32_t><<<(unsigned)top_blocks, 256, 0, st>>>(
          out, out, nprimes, prime_base, log_n, tw, info, 0);
      HEFV_LAUNCH_CHECK("k_ntt32_top");
    }
  }
  return 0;
}

template <int LOGN, int LOGE, class M>
static int launch_one(bool fwd, const typename M::T* in, typename M::T* out, int64_t batch,
                      int nprimes, int prime_base, int natural, const typename M::Tw* tw,
                      const typename InfoOf<M>::I* info, cudaStream_t st, int bcast,
                      const uint32_t* twm) {
  typedef Geo<LOGN, LOGE> G_;
  const size_t smem = (size_t)spad_size(G_::N) * sizeof(typename M::T);
  const int64_t total = batch * nprimes;
  if (total <= 0) return 0;
  if constexpr (sizeof(typename M::T) == 4 && LOGN >= 10 && LOGN <= 14 && LOGE == 4) {
    // twiddles of the 32-bit set: fwd and inverse tables have the same type
    if (!natural && !bcast)
      return launch_b32<LOGN>(fwd, reinterpret_cast<const uint32_t*>(in),
                              reinterpret_cast<uint32_t*>(out), batch, nprimes, prime_base,
                              reinterpret_cast<const uint2*>(tw),
                              reinterpret_cast<const Prime32Info*>(info), st, twm);
  }
  if constexpr (sizeof(typename M::T) == 8 && LOGN == 14 && LOGE == 4) {
    if (!natural && ntt64_split(LOGN, fwd))
      return launch_split64(LOGN, fwd, reinterpret_cast<const uint64_t*>(in),
                            reinterpret_cast<uint64_t*>(out), batch, nprimes, prime_base,
                            reinterpret_cast<const ulonglong2*>(tw),
                            reinterpret_cast<const Prime64Info*>(info), st, bcast);
  }
  if constexpr (sizeof(typename M::T) == 8 && LOGN >= 10 && LOGN <= 14 && LOGE == 4) {
    const int mode = ntt64_mode(LOGN, fwd);
    if (!natural && mode > 0)
      return launch_b64<LOGN>(fwd, reinterpret_cast<const uint64_t*>(in),
                              reinterpret_cast<uint64_t*>(out), batch, nprimes, prime_base,
                              reinterpret_cast<const ulonglong2*>(tw),
                              reinterpret_cast<const Prime64Info*>(info), st, false, bcast);
  }
  if (total > 0x7fffffff) return fail("ntt: batch too large");
  if (fwd) {
    auto kern = k_ntt_fwd<LOGN, LOGE, M>;
    HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)total, G_::NT, smem, st>>>(in, out, nprimes, prime_base, natural, tw, info,
                                                bcast);
  } else {
    auto kern = k_ntt_inv<LOGN, LOGE, M>;
    HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)total, G_::NT, smem, st>>>(in, out, nprimes, prime_base, natural, tw, info);
  }
  HEFV_LAUNCH_CHECK("ntt kernel launch");
  return 0;
}

template <class M>
static int dispatch(int log_n, bool fwd, const typename M::T* in, typename M::T* out,
                    int64_t batch, int nprimes, int prime_base, int natural,
                    const typename M::Tw* tw, const typename InfoOf<M>::I* info, cudaStream_t st,
                    int bcast = 0, const uint32_t* twm = nullptr) {
#define HEFV_CASE(L) \
  case L:            \
    return launch_one<L, 4, M>(fwd, in, out, batch, nprimes, prime_base, natural, tw, info, st, bcast, twm);
  switch (log_n) {
    case 1:
      return launch_one<1, 1, M>(fwd, in, out, batch, nprimes, prime_base, natural, tw, info, st, bcast, twm);
    case 2:
      return launch_one<2, 2, M>(fwd, in, out, batch, nprimes, prime_base, natural, tw, info, st, bcast, twm);
    case 3:
      return launch_one<3, 3, M>(fwd, in, out, batch, nprimes, prime_base, natural, tw, info, st, bcast, twm);
    HEFV_CASE(4)
    HEFV_CASE(5)
    HEFV_CASE(6)
    HEFV_CASE(7)
    HEFV_CASE(8)
    HEFV_CASE(9)
    HEFV_CASE(10)
    HEFV_CASE(11)
    HEFV_CASE(12)
    HEFV_CASE(13)
    HEFV_CASE(14)
    default:
      break;
  }
#undef HEFV_CASE
  if constexpr (sizeof(typename M::T) == 4) {
    if (log_n == 15)
      return launch_one<15, 5, M>(fwd, in, out, batch, nprimes, prime_base, natural, tw, info, st, bcast, twm);
  }
  return -100;  // not handled by the CTA-resident path
}

}  // namespace hefv

using namespace hefv;

int hefv_ntt64_large(hefv_ctx* c, bool fwd, const uint64_t* in, uint64_t* out, int64_t batch,
                     int nprimes, int prime_base, int natural, cudaStream_t st, int bcast = 0);
int hefv_ntt32_large(hefv_ctx* c, bool fwd, const uint32_t* in, uint32_t* out, int64_t batch,
                     int nprimes, int prime_base, int natural, cudaStream_t st);

// Pointwise products of canonical residues (NttPrime.negacyclic_mul's
// middle step, ntt.py:226-227): element e of row (b, i) under prime
// prime_base + i.
__global__ void k_pointwise32(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                              uint32_t* __restrict__ out, int64_t total, int log_n, int nprimes,
                              int prime_base, const Prime32Info* __restrict__ info) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)((e >> log_n) % nprimes);
    const Prime32Info inf = info[prime_base + i];
    out[e] = barrett62((uint64_t)a[e] * b[e], inf.p, inf.mu);
  }
}
__global__ void k_pointwise64(const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                              uint64_t* __restrict__ out, int64_t total, int log_n, int nprimes,
                              int prime_base, const Prime64Info* __restrict__ info) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)((e >> log_n) % nprimes);
    out[e] = mulmod64(a[e], b[e], info[prime_base + i].p);
  }
}

extern "C" {

int hefv_ntt_fwd32(hefv_ctx* c, const uint32_t* in, uint32_t* out, int64_t batch,
                   int32_t nprimes, int32_t prime_base, int32_t natural, void* stream) {
  if (!c) return fail("ntt_fwd32: null context");
  if (nprimes < 1 || prime_base < 0 || prime_base + nprimes > c->n32)
    return fail("ntt_fwd32: prime range outside the context");
  int r = dispatch<Mod32>(c->log_n, true, in, out, batch, nprimes, prime_base, natural, c->d_tw32,
                          c->d_info32, as_stream(stream), 0, c->d_twm32);
  if (r == -100) return hefv_ntt32_large(c, true, in, out, batch, nprimes, prime_base, natural,
                                         as_stream(stream));
  return r;
}

int hefv_ntt_inv32(hefv_ctx* c, const uint32_t* in, uint32_t* out, int64_t batch,
                   int32_t nprimes, int32_t prime_base, int32_t natural, void* stream) {
  if (!c) return fail("ntt_inv32: null context");
  if (nprimes < 1 || prime_base < 0 || prime_base + nprimes > c->n32)
    return fail("ntt_inv32: prime range outside the context");
  int r = dispatch<Mod32>(c->log_n, false, in, out, batch, nprimes, prime_base, natural,
                          c->d_itw32, c->d_info32, as_stream(stream), 0, c->d_itwm32);
  if (r == -100) return hefv_ntt32_large(c, false, in, out, batch, nprimes, prime_base, natural,
                                         as_stream(stream));
  return r;
}

int hefv_ntt_fwd64(hefv_ctx* c, const uint64_t* in, uint64_t* out, int64_t batch,
                   int32_t nprimes, int32_t prime_base, int32_t natural, void* stream) {
  if (!c) return fail("ntt_fwd64: null context");
  if (nprimes < 1 || prime_base < 0 || prime_base + nprimes > c->n64)
    return fail("ntt_fwd64: prime range outside the context");
  int r = dispatch<Mod64>(c->log_n, true, in, out, batch, nprimes, prime_base, natural, c->d_tw64,
                          c->d_info64, as_stream(stream));
  if (r == -100)
    return hefv_ntt64_large(c, true, in, out, batch, nprimes, prime_base, natural,
                            as_stream(stream));
  return r;
}

int hefv_ntt_inv64(hefv_ctx* c, const uint64_t* in, uint64_t* out, int64_t batch,
                   int32_t nprimes, int32_t prime_base, int32_t natural, void* stream) {
  if (!c) return fail("ntt_inv64: null context");
  if (nprimes < 1 || prime_base < 0 || prime_base + nprimes > c->n64)
    return fail("ntt_inv64: prime range outside the context");
  int r = dispatch<Mod64>(c->log_n, false, in, out, batch, nprimes, prime_base, natural,
                          c->d_itw64, c->d_info64, as_stream(stream));
  if (r == -100)
    return hefv_ntt64_large(c, false, in, out, batch, nprimes, prime_base, natural,
                            as_stream(stream));
  return r;
}

int hefv_pointwise_mul(hefv_ctx* c, int32_t wide, const void* a, const void* b, void* out,
                       int64_t batch, int32_t nprimes, int32_t prime_base, void* stream) {
  if (!c) return fail("pointwise_mul: null context");
  const int nset = wide ? c->n64 : c->n32;
  if (nprimes < 1 || prime_base < 0 || prime_base + nprimes > nset)
    return fail("pointwise_mul: prime range outside the context");
  if (batch <= 0) return 0;
  const int64_t total = batch * nprimes * (int64_t)c->n;
  const unsigned grid = (unsigned)((total + 255) / 256 < 148 * 64 ? (total + 255) / 256 : 148 * 64);
  if (wide)
    k_pointwise64<<<grid, 256, 0, as_stream(stream)>>>(
        static_cast<const uint64_t*>(a), static_cast<const uint64_t*>(b),
        static_cast<uint64_t*>(out), total, c->log_n, nprimes, prime_base, c->d_info64);
  else
    k_pointwise32<<<grid, 256, 0, as_stream(stream)>>>(
        static_cast<const uint32_t*>(a), static_cast<const uint32_t*>(b),
        static_cast<uint32_t*>(out), total, c->log_n, nprimes, prime_base, c->d_info32);
  HEFV_LAUNCH_CHECK("k_pointwise");
  return 0;
}

}  // extern "C"

// Forward transforms (device order) of `rows` input rows under every 64-bit
// prime of the context: out[r][j] = NTT_j(in[r] mod p_j).  Internal (the
// 64-bit key switch reads its digit rows this way instead of materialising
// L reduced copies).
int hefv_ntt64_fwd_rows(hefv_ctx* c, const uint64_t* in, uint64_t* out, int64_t rows,
                        cudaStream_t st) {
  int r = dispatch<Mod64>(c->log_n, true, in, out, rows, c->n64, 0, 0, c->d_tw64, c->d_info64, st,
                          1);
  if (r == -100) return hefv_ntt64_large(c, true, in, out, rows, c->n64, 0, 0, st, 1);
  return r;
}

// ---------------------------------------------------------------------------
// 64-bit primes, N in {2^15, 2^16}: two CTA-resident passes through HBM.
// Pass A (stages [0, S)) treats the polynomial as 2^S columns-interleaved
// sub-problems: CTA c handles the 2^S elements {c' + e * (N >> S)} for a
// group of consecutive columns; pass B (stages [S, LOGN)) handles contiguous
// blocks of N >> S elements.  Both passes use the same twiddle indexing as
// the single-CTA transform, so results are identical.
// ---------------------------------------------------------------------------
namespace hefv {

__global__ void k_permute_bitrev64(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                   int log_n, int64_t total) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= total) return;
  const int64_t n = 1ll << log_n;
  const int64_t poly = gid >> log_n;
  const int i = (int)(gid & (n - 1));
  out[poly * n + brev_n(i, log_n)] = in[gid];
}

}  // namespace hefv

// ---------------------------------------------------------------------------
// 64-bit primes, N in {2^15, 2^16}: one thread-block CLUSTER per polynomial.
// CL = N / 2^14 CTAs of 1024 threads x 16 words; each CTA owns a 2^14-word
// tile (139 KB) of the polynomial.  The transform is the single-CTA one
// (ntt.cuh) run over the cluster's CL*1024 threads ("gtid"): its first
// radix-16 pass spans the whole polynomial, so exchange 0 goes through
// distributed shared memory (st.shared::cluster into the owner CTA's tile,
// bracketed by cluster barriers); every later pass and exchange stays inside
// one CTA's contiguous 2^14-word block, exactly as in the 2^14 transform.
// One HBM read and one HBM write per polynomial (the radix-pass fallback
// below makes four round trips).  Same twiddle tables and butterflies, so
// the limbs are identical to the other paths.
// ---------------------------------------------------------------------------
namespace hefv {

template <int LOGN, class M>
struct Cl64 {
  static constexpr int CL = 1 << (LOGN - 14);  // CTAs per cluster
  static constexpr int LOCAL = 1 << 14;        // words per CTA tile
  // every exchange pads with ratio 1/16 (xpad_k / xpad_s), so a CTA's block
  // [r LOCAL, (r+1) LOCAL) starts at padded address r * LP
  static constexpr int LP = LOCAL + LOCAL / 16;
  static constexpr size_t smem = (size_t)((spad_size(LOCAL) + 3) & ~3) * sizeof(typename M::T);
};

__device__ __forceinline__ void dsmem_st(uint32_t addr, uint64_t v) { dsmem_st64(addr, v); }
__device__ __forceinline__ void dsmem_st(uint32_t addr, uint32_t v) { dsmem_st32(addr, v); }

template <int LOGN, class M, class TIn>
__global__ void __cluster_dims__(1 << (LOGN - 14), 1, 1) __launch_bounds__(1024, 1)
    k_ntt_cl_fwd(const TIn* __restrict__ in, typename M::T* __restrict__ out, int nprimes,
                 int prime_base, const typename M::Tw* __restrict__ tw_all,
                 const typename InfoOf<M>::I* __restrict__ info, int bcast) {
  typedef Geo<LOGN, 4> G_;
  typedef Cl64<LOGN, M> C_;
  typedef typename M::T T;
  constexpr int E = 16, NT = G_::NT, LP = C_::LP;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const int tid = threadIdx.x;
  const int r = (int)cluster_ctarank();
  const int gtid = r * 1024 + tid;
  const size_t poly = blockIdx.x / C_::CL;
  const int pi = prime_base + (int)(poly % nprimes);
  const auto* ip = info + pi;
  const M md = make_mod(*ip);
  const typename M::Tw* tw = tw_all + (size_t)pi * G_::N;
  const TIn* src = in + (bcast ? poly / nprimes : poly) * G_::N;
  T* dst = out + poly * G_::N;
  T x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = cl_in(src[gtid + e * NT], *ip);
  fwd_full_pass<LOGN, 4, M>(md, x, 0, gtid, tw);
  cluster_sync_all();  // every CTA of the cluster is running (its tile may be written)
  {
    constexpr int K = xpad_k(LOGN, 4, 0), S = xpad_s(LOGN, 4, 0);
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int owner = e / (E / C_::CL);  // element gtid + e NT lives in block `owner`
      const int a = xaddr_full<LOGN, 4>(0, gtid, e, K, S) - owner * LP;
      dsmem_st(dsmem_map(base + (uint32_t)(sizeof(T) * a), (uint32_t)owner), x[e]);
    }
    cluster_sync_all();
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = sm[xaddr_full<LOGN, 4>(1, gtid, e, K, S) - r * LP];
  }
#pragma unroll
  for (int pass = 1; pass < G_::NFULL; ++pass) {
    fwd_full_pass<LOGN, 4, M>(md, x, pass, gtid, tw);
    group_sync<10>(tid, LOGN - (pass + 1) * 4);
    const int K = xpad_k(LOGN, 4, pass), S = xpad_s(LOGN, 4, pass);
#pragma unroll
    for (int e = 0; e < E; ++e) sm[xaddr_full<LOGN, 4>(pass, gtid, e, K, S) - r * LP] = x[e];
    group_sync<10>(tid, LOGN - (pass + 1) * 4);
    if (pass + 1 < G_::NFULL) {
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = sm[xaddr_full<LOGN, 4>(pass + 1, gtid, e, K, S) - r * LP];
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = sm[xaddr_row<LOGN, 4>(gtid, e, K, S) - r * LP];
    }
  }
  fwd_last_pass<LOGN, 4, M>(md, x, gtid, tw);
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = md.canon4(x[e]);
  store_row_vec<LOGN, 4, T>(dst, gtid, x);
}

template <int LOGN, class M>
__global__ void __cluster_dims__(1 << (LOGN - 14), 1, 1) __launch_bounds__(1024, 1)
    k_ntt_cl_inv(const typename M::T* __restrict__ in, typename M::T* __restrict__ out,
                 int nprimes, int prime_base, const typename M::Tw* __restrict__ itw_all,
                 const typename InfoOf<M>::I* __restrict__ info, int /*bcast*/) {
  typedef Geo<LOGN, 4> G_;
  typedef Cl64<LOGN, M> C_;
  typedef typename M::T T;
  constexpr int E = 16, NT = G_::NT, LP = C_::LP;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  const int tid = threadIdx.x;
  const int r = (int)cluster_ctarank();
  const int gtid = r * 1024 + tid;
  const size_t poly = blockIdx.x / C_::CL;
  const int pi = prime_base + (int)(poly % nprimes);
  const auto* ip = info + pi;
  const M md = make_mod(*ip);
  const typename M::Tw* itw = itw_all + (size_t)pi * G_::N;
  const T* src = in + poly * G_::N;
  T* dst = out + poly * G_::N;
  T x[E];
  load_row_vec<LOGN, 4, T>(src, gtid, x);
  inv_last_pass<LOGN, 4, M>(md, x, gtid, itw, ip->ninv, ip->wn);
#pragma unroll
  for (int pass = G_::NFULL - 1; pass >= 1; --pass) {
    const int K = xpad_k(LOGN, 4, pass), S = xpad_s(LOGN, 4, pass);
    if (pass == G_::NFULL - 1) {
#pragma unroll
      for (int e = 0; e < E; ++e) sm[xaddr_row<LOGN, 4>(gtid, e, K, S) - r * LP] = x[e];
    } else {
      group_sync<10>(tid, LOGN - (pass + 2) * 4);
#pragma unroll
      for (int e = 0; e < E; ++e) sm[xaddr_full<LOGN, 4>(pass + 1, gtid, e, K, S) - r * LP] = x[e];
    }
    group_sync<10>(tid, LOGN - (pass + 1) * 4);
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = sm[xaddr_full<LOGN, 4>(pass, gtid, e, K, S) - r * LP];
    inv_full_pass<LOGN, 4, M>(md, x, pass, gtid, itw, ip->ninv, ip->wn);
  }
  // exchange 0 (pass-1 layout -> pass-0 layout) through DSMEM: element i goes
  // to the CTA whose threads read it in pass 0, r' = (i mod NT) / 1024, at the
  // local index (i mod 1024) + (i / NT) * 1024 of that CTA's tile
  cluster_sync_all();  // every CTA has finished reading its own tile
  {
    constexpr int K = xpad_k(LOGN, 4, 0), S = xpad_s(LOGN, 4, 0);
    constexpr int TSH1 = LOGN - 8;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    const int G1 = gtid >> TSH1, L1 = gtid & ((1 << TSH1) - 1);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = (G1 << (LOGN - 4)) + L1 + (e << TSH1);
      const int owner = (i & (NT - 1)) >> 10;
      const int li = (i & 1023) + ((i >> (LOGN - 4)) << 10);
      dsmem_st(dsmem_map(base + (uint32_t)(sizeof(T) * (li + K * (li >> S))), (uint32_t)owner),
               x[e]);
    }
    cluster_sync_all();
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int li = tid + (e << 10);
      x[e] = sm[li + K * (li >> S)];
    }
  }
  inv_full_pass<LOGN, 4, M>(md, x, 0, gtid, itw, ip->ninv, ip->wn);
#pragma unroll
  for (int e = 0; e < E; ++e) dst[gtid + e * NT] = md.subp(x[e]);
}

template <int LOGN, class M, class TIn>
static int launch_cl(bool fwd, const TIn* in, typename M::T* out, int64_t total_polys,
                     int nprimes, int prime_base, const typename M::Tw* tw,
                     const typename InfoOf<M>::I* info, cudaStream_t st, int bcast) {
  typedef Cl64<LOGN, M> C_;
  if (total_polys * C_::CL > 0x7fffffff) return fail("ntt: batch too large");
  if (fwd) {
    auto kern = k_ntt_cl_fwd<LOGN, M, TIn>;
    HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C_::smem));
    kern<<<(unsigned)(total_polys * C_::CL), 1024, C_::smem, st>>>(in, out, nprimes, prime_base, tw,
                                                                   info, bcast);
  } else {
    if constexpr (sizeof(TIn) == sizeof(typename M::T)) {
      auto kern = k_ntt_cl_inv<LOGN, M>;
      HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C_::smem));
      kern<<<(unsigned)(total_polys * C_::CL), 1024, C_::smem, st>>>(
          reinterpret_cast<const typename M::T*>(in), out, nprimes, prime_base, tw, info, bcast);
    } else {
      return fail("ntt: inverse input must have the word type");
    }
  }
  HEFV_LAUNCH_CHECK("k_ntt_cl");
  return 0;
}


}  // namespace hefv

int hefv_ntt64_large(hefv_ctx* c, bool fwd, const uint64_t* in, uint64_t* out, int64_t batch,
                     int nprimes, int prime_base, int natural, cudaStream_t st, int bcast) {
  const int log_n = c->log_n;
  const int64_t n = c->n;
  const int64_t total_polys = batch * nprimes;
  if (total_polys <= 0) return 0;
  if (bcast && !(log_n == 15 || log_n == 16))
    return fail("ntt64: broadcast input rows need N = 2^15 or 2^16");
  if (log_n == 15 || log_n == 16) {
    auto run = [&](const uint64_t* a, uint64_t* b) {
      const ulonglong2* tw = fwd ? c->d_tw64 : c->d_itw64;
      return launch_split64(log_n, fwd, a, b, batch, nprimes, prime_base, tw, c->d_info64, st,
                            bcast);
    };
    const int64_t tot = total_polys * n;
    if (!natural) return run(in, out);
    if (fwd) {
      // device order into out, then permute into natural order through a temporary
      int rc = run(in, out);
      if (rc) return rc;
      uint64_t* tmp = nullptr;
      HEFV_CUDA(cudaMallocAsync(&tmp, tot * 8, st));
      k_permute_bitrev64<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(out, tmp, log_n, tot);
      HEFV_LAUNCH_CHECK("ntt64 permute");
      HEFV_CUDA(cudaMemcpyAsync(out, tmp, tot * 8, cudaMemcpyDeviceToDevice, st));
      HEFV_CUDA(cudaFreeAsync(tmp, st));
      return 0;
    }
    // natural -> device order into out, then the inverse in place (every CTA
    // of k_ntt64_sub loads its sub-block before it stores, k_ntt64_top is
    // thread-local)
    k_permute_bitrev64<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(in, out, log_n, tot);
    HEFV_LAUNCH_CHECK("ntt64 permute");
    return run(out, out);
  }
  return fail("ntt64_large: N must be 2^15 or 2^16");
}

// 32-bit primes at N = 2^16: the cluster transform (device order only).
int hefv_ntt32_large(hefv_ctx* c, bool fwd, const uint32_t* in, uint32_t* out, int64_t batch,
                     int nprimes, int prime_base, int natural, cudaStream_t st) {
  if (c->log_n != 16) return fail("ntt32: unsupported ring dimension");
  if (natural) return fail("ntt32: N = 2^16 runs in device order only");
  return launch_split32<2, uint32_t>(fwd, in, out, batch, nprimes, prime_base,
                                     fwd ? c->d_tw32 : c->d_itw32, c->d_info32,
                                     fwd ? c->d_twm32 : c->d_itwm32, st, 0);
}

// Forward transforms (device order) of u64 rows (< 2^62) under the 32-bit
// primes [prime_base, prime_base + nprimes): out[r][t] = NTT_t(in[r] mod a_t).
// Internal: the aux-basis 64-bit key switch feeds its digits through this.
int hefv_ntt32_fwd_rows64(hefv_ctx* c, const uint64_t* in, uint32_t* out, int64_t rows,
                          int nprimes, int prime_base, cudaStream_t st) {
  const int64_t total = rows * nprimes;
  if (total <= 0) return 0;
  if (total > 0x7fffffff) return fail("ntt32_rows64: batch too large");
  switch (c->log_n) {
#define HEFV_R64(L)                                                                          \
  case L: {                                                                                  \
    typedef Geo<L, 4> G_;                                                                    \
    const size_t smem = (size_t)spad_size(G_::N) * 4;                                        \
    auto kern = k_ntt_fwd<L, 4, Mod32, uint64_t>;                                            \
    HEFV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kern<<<(unsigned)total, G_::NT, smem, st>>>(in, out, nprimes, prime_base, 0, c->d_tw32,  \
                                                c->d_info32, 1);                             \
    HEFV_LAUNCH_CHECK("k_ntt_fwd rows64");                                                   \
    return 0;                                                                                \
  }
    HEFV_R64(10)
    HEFV_R64(11)
    HEFV_R64(12)
    HEFV_R64(13)
    HEFV_R64(14)
#undef HEFV_R64
    case 15:  // (the split form measured equal here: its outer pass is one stage per HBM trip)
      return launch_cl<15, Mod32, uint64_t>(true, in, out, total, nprimes, prime_base, c->d_tw32,
                                            c->d_info32, st, 1);
    case 16:
      return launch_split32<2, uint64_t>(true, in, out, rows, nprimes, prime_base, c->d_tw32,
                                         c->d_info32, c->d_twm32, st, 1);
    default:
      return fail("ntt32_rows64: ring dimension outside 2^10..2^16");
  }
}
