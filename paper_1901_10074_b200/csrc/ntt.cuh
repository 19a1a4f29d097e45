// CTA-resident negacyclic NTT (one polynomial of N = 2^LOGN words per CTA).
//
// Replaces NttPrime.fwd / NttPrime.inv (reference ntt.py:216-224, kernel
// ntt.py:28-61).  Same mathematical transform -- evaluations of a(x) at the
// odd powers psi^(2k+1), with psi = g^((p-1)/2N) for the smallest generator g
// (ntt.py:155-156) -- computed the B200 way:
//   * the psi twist is merged into the twiddles (Cooley-Tukey with
//     psi^bitrev(i) tables, Gentleman-Sande with psi^-bitrev(i) and N^{-1}
//     folded into the last stage), so there is no separate twist pass;
//   * the transform runs as radix-2^LOGE register passes: each thread holds
//     E = 2^LOGE words and performs LOGE butterfly stages in registers, and
//     passes exchange through one padded shared-memory tile;
//   * the forward output is in bit-reversed evaluation order ("device NTT
//     order"): dev[i] = ref_fwd[bitrev(i)].  Pointwise products are order
//     agnostic, so keys / plaintexts are permuted once on upload and every
//     coefficient-domain limb is bit-identical to the reference's.
//
// Register layouts (tid in [0, NT), NT = N / E):
//   * "column" layout (pass 0 input, inverse output): element tid + e*NT.
//     Global loads/stores in this layout are fully coalesced.
//   * "row" layout (forward output, inverse input): row_index(tid, e) --
//     blocks of 2^RLAST consecutive words, block b * NT + tid for register
//     block b -> 128-bit vector loads/stores, conflict-free tile accesses.
#pragma once
#include "modarith.cuh"

#ifndef HEFV_DIAG
// Timing diagnostics only (the results are wrong): 1 no shared-memory exchanges,
// 2 no group barriers, 8 no output (k_ntt32_b), 16 no input (k_ntt32_b).  Built
// with tools/build_variant.sh; they priced the parts of a transform.
#define HEFV_DIAG 0
#endif

namespace hefv {

// Shared-tile address map: an XOR swizzle of the low 5 bits with bits
// [LOGE, LOGE + 5).  With the register layouts below it makes every exchange
// of every supported (N, E) conflict-free (checked exhaustively on the host),
// and, being a bijection on [0, N), needs no padding words.
template <int LOGE>
__device__ __forceinline__ int swz(int x) { return x + (x >> 4); }
__device__ __forceinline__ int spad(int x) { return x + (x >> 4); }
__host__ __device__ constexpr int spad_size(int n) { return n + (n >> 4) + 1; }

template <int LOGN, int LOGE>
struct Geo {
  static constexpr int N = 1 << LOGN;
  static constexpr int E = 1 << LOGE;
  static constexpr int NT = N >> LOGE;
  static constexpr int NFULL = (LOGN - 1) / LOGE;       // full radix-E passes
  static constexpr int RLAST = LOGN - LOGE * NFULL;     // stages of the last pass (1..LOGE)
  static constexpr int BLK = E >> RLAST;                // last-pass blocks per thread
  static_assert(LOGN > LOGE || (LOGN == LOGE), "N must be >= E");
};

// Index of register e of thread tid in the "row" layout (forward output /
// inverse input): E consecutive words per thread (the last pass's blocks of
// 2^RLAST words are contiguous per thread), so every exchange after pass 0
// stays inside a warp or a small warp group, and global accesses are
// 128-bit vectors.
template <int LOGN, int LOGE>
__device__ __forceinline__ int row_index(int tid, int e) {
  return (tid << LOGE) + e;
}

// Load a contiguous run of `count` (<= MAXC, compile-time after unrolling)
// twiddles with 16-byte accesses where possible.
template <class Tw, int MAXC>
__device__ __forceinline__ void load_tw_run(const Tw* __restrict__ p, Tw* out, const int count) {
  if (sizeof(Tw) == 4 && count % 4 == 0) {  // single-word (Montgomery) twiddles
    const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int i = 0; i < MAXC / 4; ++i) {
      if (4 * i < count) {
        const uint4 v = q[i];
        out[4 * i] = *reinterpret_cast<const Tw*>(&v.x);
        out[4 * i + 1] = *reinterpret_cast<const Tw*>(&v.y);
        out[4 * i + 2] = *reinterpret_cast<const Tw*>(&v.z);
        out[4 * i + 3] = *reinterpret_cast<const Tw*>(&v.w);
      }
    }
  } else if (sizeof(Tw) == 8 && count % 2 == 0) {
    const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int i = 0; i < MAXC / 2; ++i) {
      if (2 * i < count) {
        const uint4 v = q[i];
        out[2 * i] = *reinterpret_cast<const Tw*>(&v.x);
        out[2 * i + 1] = *reinterpret_cast<const Tw*>(&v.z);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < MAXC; ++i)
      if (i < count) out[i] = p[i];
  }
}

// ---- forward (Cooley-Tukey, natural -> bit-reversed) ----------------------

template <int LOGN, int LOGE, class M>
__device__ __forceinline__ void fwd_full_pass(const M& md, typename M::T* x, int pass, int tid,
                                              const typename M::Tw* __restrict__ tw,
                                              const int base = 1) {
  typedef Geo<LOGN, LOGE> G_;
  const int s0 = pass * LOGE;
  const int tsh = LOGN - s0 - LOGE;  // log2 of the element stride T
  const int G = tid >> tsh;
#pragma unroll
  for (int l = 0; l < LOGE; ++l) {
    const int half = G_::E >> (l + 1);
    if constexpr (sizeof(typename M::Tw) > 8) {
      // 64-bit primes: one 16-byte twiddle per butterfly group, loaded where
      // used (an array of 16-byte pairs would be placed in local memory)
      const typename M::Tw* twb = tw + (base << (s0 + l)) + (G << l);
#pragma unroll
      for (int u = 0; u < (1 << l); ++u) {
        const typename M::Tw wu = twb[u];
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) {
          const int e = u * 2 * half + e0;
          md.ct(x[e], x[e + half], wu);
        }
      }
    } else {
      // the 2^l twiddles of this stage are contiguous: 16-byte loads
      typename M::Tw w[1 << (LOGE - 1)];
      load_tw_run<typename M::Tw, (1 << (LOGE - 1))>(tw + (base << (s0 + l)) + (G << l), w, 1 << l);
#pragma unroll
      for (int u = 0; u < (1 << l); ++u) {
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) {
          const int e = u * 2 * half + e0;
          md.ct(x[e], x[e + half], w[u]);
        }
      }
    }
  }
}

template <int LOGN, int LOGE, class M>
__device__ __forceinline__ void fwd_last_pass(const M& md, typename M::T* x, int tid,
                                              const typename M::Tw* __restrict__ tw,
                                              const typename M::Tw* __restrict__ tw_hi = nullptr,
                                              int split_log = 31, const int base = 1) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int R = G_::RLAST;
  constexpr int s0 = LOGN - R;
  constexpr int BLK = G_::BLK;
  // the thread owns blocks tid*BLK .. tid*BLK+BLK-1, so at stage l its
  // twiddles are one contiguous run of BLK * 2^l table entries
#pragma unroll
  for (int l = 0; l < R; ++l) {
    const int half = (1 << R) >> (l + 1);
    // stages whose table slice lies below 2^split_log read `tw` (e.g. a shared
    // copy), the others `tw_hi` (global, through L1)
    const typename M::Tw* src = (tw_hi == nullptr || s0 + l + 1 <= split_log) ? tw : tw_hi;
    if constexpr (sizeof(typename M::Tw) > 8) {
      const typename M::Tw* twb = src + (base << (s0 + l)) + ((tid * BLK) << l);
#pragma unroll
      for (int b = 0; b < BLK; ++b) {
        typename M::T* xb = x + b * (1 << R);
#pragma unroll
        for (int u = 0; u < (1 << l); ++u) {
          const typename M::Tw wu = twb[(b << l) + u];
#pragma unroll
          for (int e0 = 0; e0 < half; ++e0) {
            const int e = u * 2 * half + e0;
            md.ct(xb[e], xb[e + half], wu);
          }
        }
      }
    } else {
      typename M::Tw w[BLK << (R - 1)];
      load_tw_run<typename M::Tw, (BLK << (R - 1))>(src + (base << (s0 + l)) + ((tid * BLK) << l),
                                                    w, BLK << l);
#pragma unroll
      for (int b = 0; b < BLK; ++b) {
        typename M::T* xb = x + b * (1 << R);
#pragma unroll
        for (int u = 0; u < (1 << l); ++u) {
#pragma unroll
          for (int e0 = 0; e0 < half; ++e0) {
            const int e = u * 2 * half + e0;
            md.ct(xb[e], xb[e + half], w[(b << l) + u]);
          }
        }
      }
    }
  }
}

// smem index of register e after full pass `pass` (its output layout)
template <int LOGN, int LOGE>
__device__ __forceinline__ int full_pass_index(int pass, int tid, int e) {
  const int s0 = pass * LOGE;
  const int tsh = LOGN - s0 - LOGE;
  const int G = tid >> tsh;
  const int L = tid & ((1 << tsh) - 1);
  return (G << (LOGN - s0)) + L + (e << tsh);
}

// ---- exchange addressing ---------------------------------------------------
// Exchange xi moves data from full-pass-xi layout to full-pass-(xi+1) (or row)
// layout through the tile with the padding map pad(x) = x + K (x >> S).
// (K, S) per exchange were chosen by an exhaustive bank simulation so that
// both the writes and the reads of every exchange are conflict-free for all
// supported (N, E).  All exchanges of one transform use the same padding
// ratio K / 2^S (1/16 for E = 16, 1/32 for E = 32): a group's element region
// (a multiple of 2^S words) then maps to the same address range in every
// exchange, which is what makes the group-scoped barriers sufficient.  The
// tile needs at most N + N/16 words.  Addresses are a per-thread base plus a
// compile-time offset per register.
__host__ __device__ constexpr int xpad_k(int LOGN, int LOGE, int xi) {
  return LOGE == 4 ? (xi == (LOGN - 1) / 4 - 1 ? 1 : 2) : 1;
}
__host__ __device__ constexpr int xpad_s(int LOGN, int LOGE, int xi) {
  return LOGE == 4 ? (xi == (LOGN - 1) / 4 - 1 ? 4 : 5) : 5;
}

template <int LOGN, int LOGE>
__device__ __forceinline__ int xaddr_full(int pass, int tid, int e, int K, int S) {
  const int s0 = pass * LOGE;
  const int tsh = LOGN - s0 - LOGE;
  const int T = 1 << tsh;
  const int G = tid >> tsh;
  const int L = tid & (T - 1);
  const int A = G << (LOGN - s0);
  int base = A + L;
  int off = e * T;
  if (K) {
    base += K * (A >> S) + (T >= (1 << S) ? K * (L >> S) : 0);
    off += T >= (1 << S) ? K * e * (T >> S) : K * ((e * T) >> S);
  }
  return base + off;
}

template <int LOGN, int LOGE>
__device__ __forceinline__ int xaddr_row(int tid, int e, int K, int S) {
  const int A = tid << LOGE;
  int base = A + (K ? K * (A >> S) : 0);
  int off = e + ((K && (1 << LOGE) >= (1 << S)) ? K * (e >> S) : 0);
  return base + off;
}

// Barrier over the group of 2^GL threads that exchange data through the
// tile: a warp-local __syncwarp when the group fits a warp, a named barrier
// (ids 1..8, one per group) for multi-warp groups, __syncthreads for the CTA.
// (GL is a compile-time constant after the pass loops are unrolled.)
template <int LOG_NT>
__device__ __forceinline__ void group_sync(int tid, const int GL) {
  if (GL >= LOG_NT) {
    __syncthreads();
  } else if (GL <= 5) {
    __syncwarp();
  } else {
    const int G = (GL > LOG_NT - 3) ? GL : LOG_NT - 3;  // at most 8 groups
    if (G >= LOG_NT) {
      __syncthreads();
    } else {
      asm volatile("bar.sync %0, %1;" ::"r"(1 + (tid >> G)), "r"(1 << G) : "memory");
    }
  }
}

// Forward transform of x (column layout in registers) -> row layout in
// registers, lazily reduced to [0, 4p).  `sm` is a padded tile of
// spad_size(N) words.  The exchange after full pass p only involves the
// 2^(LOGN - (p+1) LOGE) threads that share a pass-p region, so only the first
// exchange is CTA-wide; later ones use group / warp barriers.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// `hook` runs right after the first CTA-wide barrier of the transform, i.e.
// once every thread has consumed its input registers' source (used to
// recycle an input staging buffer).
template <int LOGN, int LOGE, class M, class Hook = NoHook, bool LAST = true>
__device__ __forceinline__ void cta_fwd(const M& md, typename M::T* x, typename M::T* sm,
                                        const typename M::Tw* __restrict__ tw,
                                        const typename M::Tw* __restrict__ tw_last = nullptr,
                                        const Hook& hook = Hook(), int split_log = 0,
                                        const int base = 1) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int LOG_NT = LOGN - LOGE;
  const int tid = threadIdx.x;
#pragma unroll
  for (int pass = 0; pass < G_::NFULL; ++pass) {
    fwd_full_pass<LOGN, LOGE, M>(md, x, pass, tid, tw, base);
    // pre-write barrier: CTA-wide before the first exchange (the tile may still
    // be read by the previous transform), group-wide afterwards
    if (pass == 0) {
      __syncthreads();
      hook();
    } else {
#if !(HEFV_DIAG & 2)
      group_sync<LOG_NT>(tid, LOGN - (pass + 1) * LOGE);
#endif
    }
#if !(HEFV_DIAG & 1)
    const int K = xpad_k(LOGN, LOGE, pass), S = xpad_s(LOGN, LOGE, pass);
#pragma unroll
    for (int e = 0; e < G_::E; ++e) sm[xaddr_full<LOGN, LOGE>(pass, tid, e, K, S)] = x[e];
#if !(HEFV_DIAG & 2)
    group_sync<LOG_NT>(tid, LOGN - (pass + 1) * LOGE);
#endif
    if (pass + 1 < G_::NFULL) {
#pragma unroll
      for (int e = 0; e < G_::E; ++e) x[e] = sm[xaddr_full<LOGN, LOGE>(pass + 1, tid, e, K, S)];
    } else {
#pragma unroll
      for (int e = 0; e < G_::E; ++e) x[e] = sm[xaddr_row<LOGN, LOGE>(tid, e, K, S)];
    }
#endif
  }
  // last pass: stages with table entries below 2^split_log from `tw`, the rest from tw_last
  // (LAST = false: the caller runs it, e.g. with another twiddle form)
  if (!LAST) return;
  if (tw_last == nullptr)
    fwd_last_pass<LOGN, LOGE, M>(md, x, tid, tw, nullptr, 31, base);
  else
    fwd_last_pass<LOGN, LOGE, M>(md, x, tid, tw, tw_last, split_log, base);
}

// ---- inverse (Gentleman-Sande, bit-reversed -> natural) -------------------

template <int LOGN, int LOGE, class M, bool SUB = false>
__device__ __forceinline__ void inv_last_pass(const M& md, typename M::T* x, int tid,
                                              const typename M::Tw* __restrict__ itw,
                                              const typename M::Tw& ninv, const typename M::Tw& wn,
                                              const int base = 1) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int R = G_::RLAST;
  constexpr int s0 = LOGN - R;
  constexpr int BLK = G_::BLK;
#pragma unroll
  for (int l = R - 1; l >= 0; --l) {
    const int half = (1 << R) >> (l + 1);
    if (s0 + l == 0 && !SUB) {
      // whole transform is one last pass (tiny N): merged N^-1 stage
#pragma unroll
      for (int b = 0; b < BLK; ++b) {
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) md.gs_last(x[b * (1 << R) + e0], x[b * (1 << R) + e0 + half], ninv, wn);
      }
      continue;
    }
    if constexpr (sizeof(typename M::Tw) > 8) {
      // 64-bit primes: twiddles loaded where used (see fwd_full_pass)
      const typename M::Tw* twb = itw + (base << (s0 + l)) + ((tid * BLK) << l);
#pragma unroll
      for (int b = 0; b < BLK; ++b) {
        typename M::T* xb = x + b * (1 << R);
#pragma unroll
        for (int u = 0; u < (1 << l); ++u) {
          const typename M::Tw wu = twb[(b << l) + u];
#pragma unroll
          for (int e0 = 0; e0 < half; ++e0) {
            const int e = u * 2 * half + e0;
            md.gs(xb[e], xb[e + half], wu);
          }
        }
      }
    } else {
      typename M::Tw w[BLK << (R - 1)];
      load_tw_run<typename M::Tw, (BLK << (R - 1))>(itw + (base << (s0 + l)) + ((tid * BLK) << l), w,
                                                    BLK << l);
#pragma unroll
      for (int b = 0; b < BLK; ++b) {
        typename M::T* xb = x + b * (1 << R);
#pragma unroll
        for (int u = 0; u < (1 << l); ++u) {
#pragma unroll
          for (int e0 = 0; e0 < half; ++e0) {
            const int e = u * 2 * half + e0;
            md.gs(xb[e], xb[e + half], w[(b << l) + u]);
          }
        }
      }
    }
  }
}

template <int LOGN, int LOGE, class M, bool SUB = false>
__device__ __forceinline__ void inv_full_pass(const M& md, typename M::T* x, int pass, int tid,
                                              const typename M::Tw* __restrict__ itw,
                                              const typename M::Tw& ninv, const typename M::Tw& wn,
                                              const int base = 1) {
  typedef Geo<LOGN, LOGE> G_;
  const int s0 = pass * LOGE;
  const int tsh = LOGN - s0 - LOGE;
  const int G = tid >> tsh;
#pragma unroll
  for (int l = LOGE - 1; l >= 0; --l) {
    const int half = G_::E >> (l + 1);
    const typename M::Tw* twb = itw + (base << (s0 + l)) + (G << l);
#pragma unroll
    for (int u = 0; u < (1 << l); ++u) {
      if (s0 + l == 0 && !SUB) {
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) {
          const int e = u * 2 * half + e0;
          md.gs_last(x[e], x[e + half], ninv, wn);
        }
      } else {
        const typename M::Tw w = twb[u];
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) {
          const int e = u * 2 * half + e0;
          md.gs(x[e], x[e + half], w);
        }
      }
    }
  }
}

// Inverse transform: x in row layout (values < 2p) -> column layout
// (natural coefficient order), values in [0, 2p).  N^{-1} is applied.
// Exchanges run from fine (warp / group) to coarse (CTA-wide).
// `itw_last` (optional): table the last pass reads instead of `itw` (e.g. the
// full-pass entries staged in shared memory as `itw`, the rest from global).
// `hook` runs right after the transform's first CTA-wide barrier (every
// thread has consumed its input registers' source by then).
// FIRST = false: the caller has run the first (register-only) pass itself,
// e.g. with another twiddle form.
// SUB = true, base = 2^S + g: the transform is sub-block g of a 2^(LOGN+S)-point
// one (table entries base << stage; its stage 0 is an ordinary butterfly, the
// N^-1 merge happens in the enclosing transform's last stage).
template <int LOGN, int LOGE, class M, class Hook = NoHook, bool FIRST = true, bool SUB = false>
__device__ __forceinline__ void cta_inv(const M& md, typename M::T* x, typename M::T* sm,
                                        const typename M::Tw* __restrict__ itw,
                                        const typename M::Tw& ninv, const typename M::Tw& wn,
                                        const typename M::Tw* __restrict__ itw_last = nullptr,
                                        const Hook& hook = Hook(), const int base = 1) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int LOG_NT = LOGN - LOGE;
  const int tid = threadIdx.x;
  if (FIRST) inv_last_pass<LOGN, LOGE, M, SUB>(md, x, tid, itw_last ? itw_last : itw, ninv, wn, base);
#pragma unroll
  for (int pass = G_::NFULL - 1; pass >= 0; --pass) {
    // group of this exchange: threads sharing a pass-`pass` region
    // this exchange is the inverse of forward exchange `pass`: same padding
    const int K = xpad_k(LOGN, LOGE, pass), S = xpad_s(LOGN, LOGE, pass);
#if HEFV_DIAG & 1
    if (pass == G_::NFULL - 1) {
      __syncthreads();
      hook();
    }
    (void)K;
    (void)S;
#else
    if (pass == G_::NFULL - 1) {
      __syncthreads();  // the tile may still be in use by a previous transform
      hook();
#pragma unroll
      for (int e = 0; e < G_::E; ++e) sm[xaddr_row<LOGN, LOGE>(tid, e, K, S)] = x[e];
    } else {
      group_sync<LOG_NT>(tid, LOGN - (pass + 2) * LOGE);
#pragma unroll
      for (int e = 0; e < G_::E; ++e) sm[xaddr_full<LOGN, LOGE>(pass + 1, tid, e, K, S)] = x[e];
    }
    group_sync<LOG_NT>(tid, LOGN - (pass + 1) * LOGE);
#pragma unroll
    for (int e = 0; e < G_::E; ++e) x[e] = sm[xaddr_full<LOGN, LOGE>(pass, tid, e, K, S)];
#endif
    inv_full_pass<LOGN, LOGE, M, SUB>(md, x, pass, tid, itw, ninv, wn, base);
  }
}

// Load / store E words of a row-layout stack (device NTT order) with 128-bit
// accesses where the block length allows it.
template <int LOGN, int LOGE>
__device__ __forceinline__ void load_row(const uint32_t* __restrict__ base, int tid, uint32_t* v) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int R = G_::RLAST;
  if constexpr ((1 << R) >= 4) {
#pragma unroll
    for (int b = 0; b < G_::BLK; ++b) {
      const uint4* p = reinterpret_cast<const uint4*>(base + row_index<LOGN, LOGE>(tid, b << R));
#pragma unroll
      for (int q = 0; q < (1 << R) / 4; ++q) {
        const uint4 w = __ldg(p + q);
        v[b * (1 << R) + 4 * q + 0] = w.x;
        v[b * (1 << R) + 4 * q + 1] = w.y;
        v[b * (1 << R) + 4 * q + 2] = w.z;
        v[b * (1 << R) + 4 * q + 3] = w.w;
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < G_::E; ++e) v[e] = __ldg(base + row_index<LOGN, LOGE>(tid, e));
  }
}

// Row-layout (E contiguous words per thread) global access, 16-byte vectors.
template <int LOGN, int LOGE, class T>
__device__ __forceinline__ void store_row_vec(T* __restrict__ base, int tid, const T* v) {
  constexpr int E = 1 << LOGE;
  constexpr int PER = 16 / sizeof(T);
  T* p = base + row_index<LOGN, LOGE>(tid, 0);
  if constexpr (E % PER == 0) {
#pragma unroll
    for (int i = 0; i < E / PER; ++i) {
      uint4 w;
      T* ws = reinterpret_cast<T*>(&w);
#pragma unroll
      for (int q = 0; q < PER; ++q) ws[q] = v[i * PER + q];
      reinterpret_cast<uint4*>(p)[i] = w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) p[e] = v[e];
  }
}
template <int LOGN, int LOGE, class T>
__device__ __forceinline__ void load_row_vec(const T* __restrict__ base, int tid, T* v) {
  constexpr int E = 1 << LOGE;
  constexpr int PER = 16 / sizeof(T);
  const T* p = base + row_index<LOGN, LOGE>(tid, 0);
  if constexpr (E % PER == 0) {
#pragma unroll
    for (int i = 0; i < E / PER; ++i) {
      const uint4 w = reinterpret_cast<const uint4*>(p)[i];
      const T* ws = reinterpret_cast<const T*>(&w);
#pragma unroll
      for (int q = 0; q < PER; ++q) v[i * PER + q] = ws[q];
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = p[e];
  }
}

// Row-layout registers (16 consecutive words per thread) -> warp-contiguous
// 16-byte chunks, through the warp's own 512-word region of the exchange tile:
// chunk c[i] of lane L is words [4 (32 i + L), +4) of the warp's 512 words, so a
// 128-bit global store of c[i] by the whole warp covers 512 contiguous bytes
// (storing the row layout directly puts each lane's 16 bytes in a different
// 64-byte run: 16 partial lines per instruction; measured 14 % of the 2^14
// forward).  Thread T's quad q sits at quad position q ^ ((T >> 1) & 3): both
// the 128-bit writes and the 128-bit reads are bank-conflict free without
// register selects.  `wbuf` must be private to the warp at this point (true
// after the forward's last exchange, which is warp-local) and 16-byte aligned.
__device__ __forceinline__ void warp_rows_to_chunks(uint32_t* wbuf, int lane, const uint32_t* x,
                                                    uint4* c) {
  const int r = (lane >> 1) & 3;
  uint4* mine = reinterpret_cast<uint4*>(wbuf + lane * 16);
  __syncwarp();  // every lane has read its exchange data out of the region
#pragma unroll
  for (int q = 0; q < 4; ++q)
    mine[q ^ r] = make_uint4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ch = i * 32 + lane;
    const int T = ch >> 2;
    c[i] = reinterpret_cast<const uint4*>(wbuf + T * 16)[(ch & 3) ^ ((T >> 1) & 3)];
  }
}
// 64-bit words: 16 consecutive words per thread are 8 quads of 16 bytes; thread
// T's quad q sits at position q ^ (T & 7).  rows -> chunks (forward output):
// chunk c[i] of lane L is bytes [16 (32 i + L), +16) of the warp's 4 KB.
__device__ __forceinline__ void warp_rows_to_chunks64(uint64_t* wbuf, int lane, const uint64_t* x,
                                                      uint4* c) {
  const int r = lane & 7;
  uint4* mine = reinterpret_cast<uint4*>(wbuf + lane * 16);
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint4 v;
    v.x = (uint32_t)x[2 * q];
    v.y = (uint32_t)(x[2 * q] >> 32);
    v.z = (uint32_t)x[2 * q + 1];
    v.w = (uint32_t)(x[2 * q + 1] >> 32);
    mine[q ^ r] = v;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int ch = i * 32 + lane;
    const int T = ch >> 3;
    c[i] = reinterpret_cast<const uint4*>(wbuf + T * 16)[(ch & 7) ^ (T & 7)];
  }
}
// chunks -> rows (inverse input): the caller loaded chunk c[i] = bytes
// [16 (32 i + L), +16) of the warp's 4 KB with coalesced 128-bit loads; `wbuf`
// must not be in use by any other warp (CTA barrier before the call).
__device__ __forceinline__ void warp_chunks_to_rows64(uint64_t* wbuf, int lane, const uint4* c,
                                                      uint64_t* x) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int ch = i * 32 + lane;
    const int T = ch >> 3;
    reinterpret_cast<uint4*>(wbuf + T * 16)[(ch & 7) ^ (T & 7)] = c[i];
  }
  __syncwarp();
  const int r = lane & 7;
  const uint4* mine = reinterpret_cast<const uint4*>(wbuf + lane * 16);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint4 v = mine[q ^ r];
    x[2 * q] = ((uint64_t)v.y << 32) | v.x;
    x[2 * q + 1] = ((uint64_t)v.w << 32) | v.z;
  }
}
// the warp's region of the tile after the last (1/16-padded) exchange
template <class T>
__device__ __forceinline__ T* warp_tile_region(T* sm, int tid) {
  return sm + (tid >> 5) * 544;
}

// Row-layout read of 16 consecutive 32-bit words per thread from SHARED
// memory (a bulk-copied staging row) without bank conflicts: plain 128-bit
// loads at a 64-byte lane stride serve 2 lanes per wavefront (4x the
// wavefronts); here lane L loads its quads rotated by r = (L >> 1) & 3, so
// every 8 lanes of an instruction hit 8 distinct 16-byte bank groups, and the
// registers are un-rotated with two conditional quad shifts (32 SELs).
__device__ __forceinline__ void load_row16_smem(const uint32_t* base, int tid, uint32_t* x) {
  const int rot = (tid >> 1) & 3;
  const uint4* p = reinterpret_cast<const uint4*>(base + (tid << 4));
  uint4 v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = p[(q + rot) & 3];  // v[q] = quad (q + rot) & 3
  // quad qq = v[(qq - rot) & 3]: rotate right by rot & 1, then by rot & 2
  const bool r1 = rot & 1, r2 = rot & 2;
  uint4 w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 a = v[q], b = v[(q + 3) & 3];
    w[q] = make_uint4(r1 ? b.x : a.x, r1 ? b.y : a.y, r1 ? b.z : a.z, r1 ? b.w : a.w);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 a = w[q], b = w[(q + 2) & 3];
    x[4 * q + 0] = r2 ? b.x : a.x;
    x[4 * q + 1] = r2 ? b.y : a.y;
    x[4 * q + 2] = r2 ? b.z : a.z;
    x[4 * q + 3] = r2 ? b.w : a.w;
  }
}

}  // namespace hefv
