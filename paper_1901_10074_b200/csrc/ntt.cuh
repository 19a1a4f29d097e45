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

namespace hefv {

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
// inverse input).  The last pass works on blocks of 2^RLAST consecutive
// words; thread tid owns blocks b * NT + tid (b < BLK), so for a fixed
// register consecutive threads touch consecutive blocks (conflict-free with
// the padded tile, 16-byte vectorisable within a block).
template <int LOGN, int LOGE>
__device__ __forceinline__ int row_index(int tid, int e) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int R = G_::RLAST;
  return ((((e >> R) * G_::NT) + tid) << R) | (e & ((1 << R) - 1));
}

// ---- forward (Cooley-Tukey, natural -> bit-reversed) ----------------------

template <int LOGN, int LOGE, class M>
__device__ __forceinline__ void fwd_full_pass(const M& md, typename M::T* x, int pass, int tid,
                                              const typename M::Tw* __restrict__ tw) {
  typedef Geo<LOGN, LOGE> G_;
  const int s0 = pass * LOGE;
  const int tsh = LOGN - s0 - LOGE;  // log2 of the element stride T
  const int G = tid >> tsh;
#pragma unroll
  for (int l = 0; l < LOGE; ++l) {
    const int half = G_::E >> (l + 1);
    const typename M::Tw* twb = tw + (1 << (s0 + l)) + (G << l);
#pragma unroll
    for (int u = 0; u < (1 << l); ++u) {
      const typename M::Tw w = twb[u];
#pragma unroll
      for (int e0 = 0; e0 < half; ++e0) {
        const int e = u * 2 * half + e0;
        md.ct(x[e], x[e + half], w);
      }
    }
  }
}

template <int LOGN, int LOGE, class M>
__device__ __forceinline__ void fwd_last_pass(const M& md, typename M::T* x, int tid,
                                              const typename M::Tw* __restrict__ tw) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int R = G_::RLAST;
  constexpr int s0 = LOGN - R;
#pragma unroll
  for (int b = 0; b < G_::BLK; ++b) {
    const int G = b * G_::NT + tid;
    typename M::T* xb = x + b * (1 << R);
#pragma unroll
    for (int l = 0; l < R; ++l) {
      const int half = (1 << R) >> (l + 1);
      const typename M::Tw* twb = tw + (1 << (s0 + l)) + (G << l);
#pragma unroll
      for (int u = 0; u < (1 << l); ++u) {
        const typename M::Tw w = twb[u];
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) {
          const int e = u * 2 * half + e0;
          md.ct(xb[e], xb[e + half], w);
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

// Forward transform of x (column layout in registers) -> row layout in
// registers, lazily reduced to [0, 4p).  `sm` is a padded tile of
// spad_size(N) words.  Caller must __syncthreads() before reusing `sm`.
template <int LOGN, int LOGE, class M>
__device__ __forceinline__ void cta_fwd(const M& md, typename M::T* x, typename M::T* sm,
                                        const typename M::Tw* __restrict__ tw,
                                        const typename M::Tw* __restrict__ tw_last = nullptr) {
  typedef Geo<LOGN, LOGE> G_;
  const int tid = threadIdx.x;
#pragma unroll
  for (int pass = 0; pass < G_::NFULL; ++pass) {
    fwd_full_pass<LOGN, LOGE, M>(md, x, pass, tid, tw);
    // exchange: write in this pass's layout, read in the next pass's layout
#pragma unroll
    for (int e = 0; e < G_::E; ++e) sm[spad(full_pass_index<LOGN, LOGE>(pass, tid, e))] = x[e];
    __syncthreads();
    if (pass + 1 < G_::NFULL) {
#pragma unroll
      for (int e = 0; e < G_::E; ++e)
        x[e] = sm[spad(full_pass_index<LOGN, LOGE>(pass + 1, tid, e))];
    } else {
#pragma unroll
      for (int e = 0; e < G_::E; ++e) x[e] = sm[spad(row_index<LOGN, LOGE>(tid, e))];
    }
    __syncthreads();
  }
  fwd_last_pass<LOGN, LOGE, M>(md, x, tid, tw_last ? tw_last : tw);
}

// ---- inverse (Gentleman-Sande, bit-reversed -> natural) -------------------

template <int LOGN, int LOGE, class M>
__device__ __forceinline__ void inv_last_pass(const M& md, typename M::T* x, int tid,
                                              const typename M::Tw* __restrict__ itw,
                                              typename M::Tw ninv, typename M::Tw wn) {
  typedef Geo<LOGN, LOGE> G_;
  constexpr int R = G_::RLAST;
  constexpr int s0 = LOGN - R;
#pragma unroll
  for (int b = 0; b < G_::BLK; ++b) {
    const int G = b * G_::NT + tid;
    typename M::T* xb = x + b * (1 << R);
#pragma unroll
    for (int l = R - 1; l >= 0; --l) {
      const int half = (1 << R) >> (l + 1);
      const typename M::Tw* twb = itw + (1 << (s0 + l)) + (G << l);
#pragma unroll
      for (int u = 0; u < (1 << l); ++u) {
#pragma unroll
        for (int e0 = 0; e0 < half; ++e0) {
          const int e = u * 2 * half + e0;
          if (s0 + l == 0) {
            md.gs_last(xb[e], xb[e + half], ninv, wn);
          } else {
            md.gs(xb[e], xb[e + half], twb[u]);
          }
        }
      }
    }
  }
}

template <int LOGN, int LOGE, class M>
__device__ __forceinline__ void inv_full_pass(const M& md, typename M::T* x, int pass, int tid,
                                              const typename M::Tw* __restrict__ itw,
                                              typename M::Tw ninv, typename M::Tw wn) {
  typedef Geo<LOGN, LOGE> G_;
  const int s0 = pass * LOGE;
  const int tsh = LOGN - s0 - LOGE;
  const int G = tid >> tsh;
#pragma unroll
  for (int l = LOGE - 1; l >= 0; --l) {
    const int half = G_::E >> (l + 1);
    const typename M::Tw* twb = itw + (1 << (s0 + l)) + (G << l);
#pragma unroll
    for (int u = 0; u < (1 << l); ++u) {
      if (s0 + l == 0) {
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
template <int LOGN, int LOGE, class M>
__device__ __forceinline__ void cta_inv(const M& md, typename M::T* x, typename M::T* sm,
                                        const typename M::Tw* __restrict__ itw,
                                        typename M::Tw ninv, typename M::Tw wn) {
  typedef Geo<LOGN, LOGE> G_;
  const int tid = threadIdx.x;
  inv_last_pass<LOGN, LOGE, M>(md, x, tid, itw, ninv, wn);
#pragma unroll
  for (int pass = G_::NFULL - 1; pass >= 0; --pass) {
    if (pass == G_::NFULL - 1) {
#pragma unroll
      for (int e = 0; e < G_::E; ++e) sm[spad(row_index<LOGN, LOGE>(tid, e))] = x[e];
    } else {
#pragma unroll
      for (int e = 0; e < G_::E; ++e)
        sm[spad(full_pass_index<LOGN, LOGE>(pass + 1, tid, e))] = x[e];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < G_::E; ++e) x[e] = sm[spad(full_pass_index<LOGN, LOGE>(pass, tid, e))];
    __syncthreads();
    inv_full_pass<LOGN, LOGE, M>(md, x, pass, tid, itw, ninv, wn);
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
      const uint4* p = reinterpret_cast<const uint4*>(base + ((b * G_::NT + tid) << R));
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

}  // namespace hefv
