// FV-layer kernels: batching encode/decode, plaintext lifting, encryption,
// the NTT-domain half of decryption, ciphertext x plaintext products, the
// layer planner's batched MAC, Galois automorphisms, switch-key generation
// and the row accumulation of layer outputs.
//
// Every kernel computes the same canonical residues as the reference CPU
// routine it replaces (cited per kernel); ordering/fusion differences are
// confined to exact modular identities (linearity of the NTT, commutativity
// of modular addition).
#include "../../include/hefv.h"
#include "internal.h"
#include "kcommon.cuh"
#include "ntt.cuh"

namespace hefv {

#define HEFV_DISPATCH_FV(log_n, FN, ...)                       \
  switch (log_n) {                                             \
    case 4:                                                    \
      return FN<4>(__VA_ARGS__);                               \
    case 5:                                                    \
      return FN<5>(__VA_ARGS__);                               \
    case 6:                                                    \
      return FN<6>(__VA_ARGS__);                               \
    case 7:                                                    \
      return FN<7>(__VA_ARGS__);                               \
    case 8:                                                    \
      return FN<8>(__VA_ARGS__);                               \
    case 9:                                                    \
      return FN<9>(__VA_ARGS__);                               \
    case 10:                                                   \
      return FN<10>(__VA_ARGS__);                              \
    case 11:                                                   \
      return FN<11>(__VA_ARGS__);                              \
    case 12:                                                   \
      return FN<12>(__VA_ARGS__);                              \
    case 13:                                                   \
      return FN<13>(__VA_ARGS__);                              \
    case 14:                                                   \
      return FN<14>(__VA_ARGS__);                              \
    default:                                                   \
      return fail("FV kernels support N = 2^4 .. 2^14 only");  \
  }

static int need_fv(const hefv_ctx* c, const char* who) {
  if (!c) return fail(std::string(who) + ": null context");
  if (!c->fv_ready) return fail(std::string(who) + ": hefv_fv_setup has not been called");
  return 0;
}

template <int LOGN>
static size_t smem32() {
  return (size_t)spad_size(1 << LOGN) * 4;
}
template <int LOGN>
static size_t smem64() {
  return (size_t)spad_size(1 << LOGN) * 8;
}

template <class K>
static int set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return check_cuda(e, "cudaFuncSetAttribute");
  }
  return 0;
}

// a * b * 2^-32 mod p, canonical (b in Montgomery form gives a * b_plain)
__device__ __forceinline__ uint32_t mulmod_mont_canon(uint32_t a, uint32_t b, const Prime32Info& inf) {
  const uint32_t r = mont_mul_lazy(a, b, inf.p, inf.pinv_neg);
  return r >= inf.p ? r - inf.p : r;
}
__device__ __forceinline__ uint32_t mulmod_small(uint32_t a, uint32_t b, const Prime32Info& inf) {
  return barrett62((uint64_t)a * b, inf.p, inf.mu);
}
__device__ __forceinline__ uint32_t addmod(uint32_t a, uint32_t b, uint32_t p) {
  uint32_t s = a + b;
  return s >= p ? s - p : s;
}
__device__ __forceinline__ uint32_t submod(uint32_t a, uint32_t b, uint32_t p) {
  return a >= b ? a - b : a + p - b;
}
__device__ __forceinline__ uint32_t small_to_mod(int v, uint32_t p) {
  return v < 0 ? (uint32_t)((int64_t)p + v) : (uint32_t)v;
}

// ---------------------------------------------------------------------------
// encode / decode (fv.py:280-289): slot s sits at evaluation index
// slot_to_ev[s]; encode = scatter + inverse t-NTT, decode = t-NTT + gather.
// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN, 4>::NT)
    k_encode(const uint64_t* __restrict__ slots, uint64_t* __restrict__ poly, int t_index,
             const int32_t* __restrict__ dev_to_slot, const ulonglong2* __restrict__ itw_all,
             const Prime64Info* __restrict__ info) {
  typedef Geo<LOGN, 4> G_;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(smraw);
  const Prime64Info inf = info[t_index];
  const Mod64 md = make_mod(inf);
  const size_t b = blockIdx.x;
  const uint64_t* src = slots + b * (G_::N / 2);
  const int tid = threadIdx.x;
  uint64_t x[G_::E];
#pragma unroll
  for (int e = 0; e < G_::E; ++e) {
    const int s = dev_to_slot[row_index<LOGN, 4>(tid, e)];
    x[e] = s >= 0 ? reduce_any(src[s], inf) : 0ull;
  }
  cta_inv<LOGN, 4, Mod64>(md, x, sm, itw_all + (size_t)t_index * G_::N, inf.ninv, inf.wn);
  uint64_t* dst = poly + b * G_::N;
#pragma unroll
  for (int e = 0; e < G_::E; ++e) dst[tid + e * G_::NT] = md.subp(x[e]);
}

template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN, 4>::NT)
    k_encode_sparse(const int32_t* __restrict__ ptr, const int32_t* __restrict__ slot_idx,
                    const uint64_t* __restrict__ vals, uint64_t* __restrict__ poly, int t_index,
                    const int32_t* __restrict__ slot_to_dev, const ulonglong2* __restrict__ itw_all,
                    const Prime64Info* __restrict__ info) {
  typedef Geo<LOGN, 4> G_;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(smraw);
  const Prime64Info inf = info[t_index];
  const Mod64 md = make_mod(inf);
  const size_t b = blockIdx.x;
  const int tid = threadIdx.x;
  for (int i = tid; i < spad_size(G_::N); i += G_::NT) sm[i] = 0ull;
  __syncthreads();
  const int lo = ptr[b], hi = ptr[b + 1];
  for (int i = lo + tid; i < hi; i += G_::NT)
    sm[spad(slot_to_dev[slot_idx[i]])] = reduce_any(vals[i], inf);
  __syncthreads();
  uint64_t x[G_::E];
#pragma unroll
  for (int e = 0; e < G_::E; ++e) x[e] = sm[spad(row_index<LOGN, 4>(tid, e))];
  __syncthreads();
  cta_inv<LOGN, 4, Mod64>(md, x, sm, itw_all + (size_t)t_index * G_::N, inf.ninv, inf.wn);
  uint64_t* dst = poly + b * G_::N;
#pragma unroll
  for (int e = 0; e < G_::E; ++e) dst[tid + e * G_::NT] = md.subp(x[e]);
}

template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN, 4>::NT)
    k_decode(const uint64_t* __restrict__ poly, uint64_t* __restrict__ slots, int t_index,
             const int32_t* __restrict__ slot_to_dev, const ulonglong2* __restrict__ tw_all,
             const Prime64Info* __restrict__ info) {
  typedef Geo<LOGN, 4> G_;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint64_t* sm = reinterpret_cast<uint64_t*>(smraw);
  const Prime64Info inf = info[t_index];
  const Mod64 md = make_mod(inf);
  const size_t b = blockIdx.x;
  const uint64_t* src = poly + b * G_::N;
  const int tid = threadIdx.x;
  uint64_t x[G_::E];
#pragma unroll
  for (int e = 0; e < G_::E; ++e) x[e] = reduce_any(src[tid + e * G_::NT], inf);
  cta_fwd<LOGN, 4, Mod64>(md, x, sm, tw_all + (size_t)t_index * G_::N);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < G_::E; ++e) sm[spad(row_index<LOGN, 4>(tid, e))] = md.canon4(x[e]);
  __syncthreads();
  uint64_t* dst = slots + b * (G_::N / 2);
  for (int s = tid; s < G_::N / 2; s += G_::NT) dst[s] = sm[spad(slot_to_dev[s])];
}

template <int LOGN>
static int run_encode(hefv_ctx* c, const uint64_t* slots, uint64_t* poly, int64_t B,
                      cudaStream_t st) {
  if (B <= 0) return 0;
  auto kern = k_encode<LOGN>;
  if (int r = set_smem(kern, smem64<LOGN>())) return r;
  kern<<<(unsigned)B, Geo<LOGN, 4>::NT, smem64<LOGN>(), st>>>(slots, poly, c->t_index,
                                                             c->d_dev_to_slot, c->d_itw64,
                                                             c->d_info64);
  HEFV_LAUNCH_CHECK("k_encode");
  return 0;
}
template <int LOGN>
static int run_encode_sparse(hefv_ctx* c, const int32_t* ptr, const int32_t* idx,
                             const uint64_t* vals, uint64_t* poly, int64_t P, cudaStream_t st) {
  if (P <= 0) return 0;
  auto kern = k_encode_sparse<LOGN>;
  if (int r = set_smem(kern, smem64<LOGN>())) return r;
  kern<<<(unsigned)P, Geo<LOGN, 4>::NT, smem64<LOGN>(), st>>>(
      ptr, idx, vals, poly, c->t_index, c->d_slot_to_dev, c->d_itw64, c->d_info64);
  HEFV_LAUNCH_CHECK("k_encode_sparse");
  return 0;
}
template <int LOGN>
static int run_decode(hefv_ctx* c, const uint64_t* poly, uint64_t* slots, int64_t B,
                      cudaStream_t st) {
  if (B <= 0) return 0;
  auto kern = k_decode<LOGN>;
  if (int r = set_smem(kern, smem64<LOGN>())) return r;
  kern<<<(unsigned)B, Geo<LOGN, 4>::NT, smem64<LOGN>(), st>>>(poly, slots, c->t_index,
                                                             c->d_slot_to_dev, c->d_tw64,
                                                             c->d_info64);
  HEFV_LAUNCH_CHECK("k_decode");
  return 0;
}

// ---------------------------------------------------------------------------
// plaintext poly mod t -> RNS stack (fv.py:291-310, fv.py:366-370)
// ---------------------------------------------------------------------------
// Residues first (one thread per coefficient, each u64 read once, the k
// residue rows written coalesced), then the persistent batched transform
// (k_ntt32_b: prime-major, twiddles staged in shared memory; in place) and,
// when asked, the Montgomery form.  A per-(prime, plaintext) CTA that read
// its twiddles from L2 ran at a third of the batched transform's rate.
static unsigned grid_for(int64_t total, int threads);

__global__ void k_plain_residues(const uint64_t* __restrict__ poly, uint32_t* __restrict__ out,
                                 int64_t B, int k, int log_n, uint64_t t, int mode,
                                 const uint32_t* __restrict__ delta,
                                 const Prime32Info* __restrict__ info) {
  const int64_t n = 1ll << log_n;
  const uint64_t half = t >> 1;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < B * n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = g >> log_n, i = g & (n - 1);
    const uint64_t m = poly[g];
    uint32_t* dst = out + b * k * n + i;
    for (int j = 0; j < k; ++j) {
      const Prime32Info inf = info[j];
      uint32_t v;
      if (mode == 0) {
        v = mulmod_small(barrett62(m, inf.p, inf.mu), delta[j], inf);  // Delta m, m uncentred
      } else if (m > half) {
        const uint32_t r = barrett62(t - m, inf.p, inf.mu);  // centred m < 0
        v = r ? inf.p - r : 0u;
      } else {
        v = barrett62(m, inf.p, inf.mu);
      }
      dst[(int64_t)j * n] = v;
    }
  }
}

template <int LOGN>
static int run_plain_to_rns(hefv_ctx* c, const uint64_t* poly, uint32_t* out, int64_t B, int mode,
                            int to_ntt, int mont, cudaStream_t st) {
  if (B <= 0) return 0;
  const int64_t total = B << LOGN;
  k_plain_residues<<<grid_for(total, 256), 256, 0, st>>>(poly, out, B, c->k, LOGN, c->t, mode,
                                                         c->d_delta, c->d_info32);
  HEFV_LAUNCH_CHECK("k_plain_residues");
  if (to_ntt)
    if (int r = hefv_ntt_fwd32(c, out, out, B, c->k, 0, 0, st)) return r;
  if (mont)
    if (int r = hefv_to_montgomery(c, out, out, B, st)) return r;
  return 0;
}

// small signed polynomial -> residues (fv.py:119-122), optionally NTT / Montgomery
template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN, Loge32<LOGN>::v>::NT)
    k_small_to_rns(const int8_t* __restrict__ small, uint32_t* __restrict__ out, int k,
                   int to_ntt, int montgomery, const uint2* __restrict__ tw_all,
                   const Prime32Info* __restrict__ info) {
  constexpr int LE = Loge32<LOGN>::v;
  typedef Geo<LOGN, LE> G_;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smraw);
  const int j = blockIdx.x;
  const size_t b = blockIdx.y;
  const Prime32Info inf = info[j];
  const Mod32 md = make_mod(inf);
  const int8_t* src = small + b * G_::N;
  uint32_t* dst = out + (b * k + j) * (size_t)G_::N;
  const int tid = threadIdx.x;
  uint32_t x[G_::E];
#pragma unroll
  for (int e = 0; e < G_::E; ++e) x[e] = small_to_mod(src[tid + e * G_::NT], inf.p);
  if (to_ntt) {
    cta_fwd<LOGN, LE, Mod32>(md, x, sm, tw_all + (size_t)j * G_::N);
#pragma unroll
    for (int e = 0; e < G_::E; ++e) {
      uint32_t v = md.canon4(x[e]);
      if (montgomery) v = mont_canon(v, inf);
      dst[row_index<LOGN, LE>(tid, e)] = v;
    }
  } else {
#pragma unroll
    for (int e = 0; e < G_::E; ++e) {
      uint32_t v = x[e];
      if (montgomery) v = mont_canon(v, inf);
      dst[tid + e * G_::NT] = v;
    }
  }
}

template <int LOGN>
static int run_small_to_rns(hefv_ctx* c, const int8_t* small, uint32_t* out, int64_t B,
                            int to_ntt, int mont, cudaStream_t st) {
  if (B <= 0) return 0;
  typedef Geo<LOGN, Loge32<LOGN>::v> G_;
  auto kern = k_small_to_rns<LOGN>;
  if (int r = set_smem(kern, smem32<LOGN>())) return r;
  dim3 grid(c->k, (unsigned)B);
  kern<<<grid, G_::NT, smem32<LOGN>(), st>>>(small, out, c->k, to_ntt, mont, c->d_tw32,
                                             c->d_info32);
  HEFV_LAUNCH_CHECK("k_small_to_rns");
  return 0;
}

// ---------------------------------------------------------------------------
// elementwise over (rows, k, N) stacks
// ---------------------------------------------------------------------------
__global__ void k_elementwise(int op, const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                              const uint32_t* __restrict__ cc, uint32_t* __restrict__ out,
                              int64_t total, int log_n, int k, int64_t b_rows, int64_t c_rows,
                              const Prime32Info* __restrict__ info) {
  const int64_t stack = (int64_t)k << log_n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / stack;
    const int64_t w = i - row * stack;
    const int j = (int)(w >> log_n);
    const Prime32Info inf = info[j];
    const uint32_t x = a[i];
    const uint32_t y = b[(row % b_rows) * stack + w];
    uint32_t r;
    if (op == 0) {
      r = addmod(x, y, inf.p);
    } else if (op == 1) {
      r = submod(x, y, inf.p);
    } else if (op == 2) {
      r = mulmod_small(x, y, inf);
    } else {
      const uint32_t z = cc[(row % c_rows) * stack + w];
      const uint32_t s = addmod(mulmod_small(x, y, inf), z, inf.p);
      r = s ? inf.p - s : 0u;
    }
    out[i] = r;
  }
}

__global__ void k_to_mont(const uint32_t* __restrict__ a, uint32_t* __restrict__ out, int64_t total,
                          int log_n, int k, const Prime32Info* __restrict__ info) {
  const int64_t stack = (int64_t)k << log_n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)((i % stack) >> log_n);
    out[i] = mont_canon(a[i], info[j]);
  }
}

static unsigned grid_for(int64_t total, int threads) {
  int64_t g = (total + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// ---------------------------------------------------------------------------
// encryption (fv.py:317-335): c0 = iNTT(NTT(u) pk0) + e1 + dm, c1 = iNTT(NTT(u) pk1) + e2
// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN, Loge32<LOGN>::v>::NT)
    k_encrypt(const uint32_t* __restrict__ pk_ntt, const int8_t* __restrict__ u,
              const int8_t* __restrict__ e1, const int8_t* __restrict__ e2,
              const uint32_t* __restrict__ dm, uint32_t* __restrict__ out, int k,
              const uint2* __restrict__ tw_all, const uint2* __restrict__ itw_all,
              const Prime32Info* __restrict__ info) {
  constexpr int LE = Loge32<LOGN>::v;
  typedef Geo<LOGN, LE> G_;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smraw);
  const int j = blockIdx.x;
  const size_t b = blockIdx.y;
  const Prime32Info inf = info[j];
  const Mod32 md = make_mod(inf);
  const int tid = threadIdx.x;
  const size_t N = G_::N;
  uint32_t xu[G_::E], y[G_::E];
#pragma unroll
  for (int e = 0; e < G_::E; ++e) xu[e] = small_to_mod(u[b * N + tid + e * G_::NT], inf.p);
  cta_fwd<LOGN, LE, Mod32>(md, xu, sm, tw_all + (size_t)j * N);
  for (int part = 0; part < 2; ++part) {
    const uint32_t* pk = pk_ntt + ((size_t)part * k + j) * N;
#pragma unroll
    for (int e = 0; e < G_::E; ++e) y[e] = mont_mul_lazy(xu[e], pk[row_index<LOGN, LE>(tid, e)], inf.p, inf.pinv_neg);
    cta_inv<LOGN, LE, Mod32>(md, y, sm, itw_all + (size_t)j * N, inf.ninv, inf.wn);
    const int8_t* er = (part == 0 ? e1 : e2) + b * N;
    uint32_t* dst = out + ((b * 2 + part) * k + j) * N;
    const uint32_t* dmr = dm + (b * k + j) * N;
#pragma unroll
    for (int e = 0; e < G_::E; ++e) {
      const int idx = tid + e * G_::NT;
      uint32_t v = addmod(md.subp(y[e]), small_to_mod(er[idx], inf.p), inf.p);
      if (part == 0) v = addmod(v, dmr[idx], inf.p);
      dst[idx] = v;
    }
    __syncthreads();
  }
}

template <int LOGN>
static int run_encrypt(hefv_ctx* c, const uint32_t* pk, const int8_t* u, const int8_t* e1,
                       const int8_t* e2, const uint32_t* dm, uint32_t* out, int64_t B,
                       cudaStream_t st) {
  if (B <= 0) return 0;
  typedef Geo<LOGN, Loge32<LOGN>::v> G_;
  auto kern = k_encrypt<LOGN>;
  if (int r = set_smem(kern, smem32<LOGN>())) return r;
  dim3 grid(c->k, (unsigned)B);
  kern<<<grid, G_::NT, smem32<LOGN>(), st>>>(pk, u, e1, e2, dm, out, c->k, c->d_tw32, c->d_itw32,
                                             c->d_info32);
  HEFV_LAUNCH_CHECK("k_encrypt");
  return 0;
}

// ---------------------------------------------------------------------------
// decryption, NTT half (fv.py:337-347): acc_j = c0 + iNTT(sum_m NTT(c_m) s^m)
// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN, Loge32<LOGN>::v>::NT)
    k_decrypt_acc(const uint32_t* __restrict__ ct, int nparts, const uint32_t* __restrict__ s_ntt,
                  const uint32_t* __restrict__ s2_ntt, uint32_t* __restrict__ acc_out, int k,
                  const uint2* __restrict__ tw_all, const uint2* __restrict__ itw_all,
                  const Prime32Info* __restrict__ info) {
  constexpr int LE = Loge32<LOGN>::v;
  typedef Geo<LOGN, LE> G_;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smraw);
  const int j = blockIdx.x;
  const size_t b = blockIdx.y;
  const Prime32Info inf = info[j];
  const Mod32 md = make_mod(inf);
  const int tid = threadIdx.x;
  const size_t N = G_::N;
  uint32_t acc[G_::E], x[G_::E];
#pragma unroll
  for (int e = 0; e < G_::E; ++e) acc[e] = 0;
  for (int m = 1; m < nparts; ++m) {
    const uint32_t* src = ct + ((b * nparts + m) * k + j) * N;
#pragma unroll
    for (int e = 0; e < G_::E; ++e) x[e] = src[tid + e * G_::NT];
    cta_fwd<LOGN, LE, Mod32>(md, x, sm, tw_all + (size_t)j * N);
    const uint32_t* sk = (m == 1 ? s_ntt : s2_ntt) + (size_t)j * N;
#pragma unroll
    for (int e = 0; e < G_::E; ++e)
      acc[e] = md.sub2p(acc[e] + mont_mul_lazy(x[e], sk[row_index<LOGN, LE>(tid, e)], inf.p, inf.pinv_neg));
    __syncthreads();
  }
  cta_inv<LOGN, LE, Mod32>(md, acc, sm, itw_all + (size_t)j * N, inf.ninv, inf.wn);
  const uint32_t* c0 = ct + ((b * nparts) * k + j) * N;
  uint32_t* dst = acc_out + (b * k + j) * N;
#pragma unroll
  for (int e = 0; e < G_::E; ++e) {
    const int idx = tid + e * G_::NT;
    dst[idx] = addmod(md.subp(acc[e]), c0[idx], inf.p);
  }
}

template <int LOGN>
static int run_decrypt_acc(hefv_ctx* c, const uint32_t* ct, int nparts, const uint32_t* s,
                           const uint32_t* s2, uint32_t* acc, int64_t B, cudaStream_t st) {
  if (B <= 0) return 0;
  typedef Geo<LOGN, Loge32<LOGN>::v> G_;
  auto kern = k_decrypt_acc<LOGN>;
  if (int r = set_smem(kern, smem32<LOGN>())) return r;
  dim3 grid(c->k, (unsigned)B);
  kern<<<grid, G_::NT, smem32<LOGN>(), st>>>(ct, nparts, s, s2, acc, c->k, c->d_tw32, c->d_itw32,
                                             c->d_info32);
  HEFV_LAUNCH_CHECK("k_decrypt_acc");
  return 0;
}

// ---------------------------------------------------------------------------
// ciphertext x plaintext (fv.py:364-375) and the planner's row MAC
// ---------------------------------------------------------------------------
// ct x pt products and the planner's row MAC, in the NTT domain: an
// elementwise Montgomery product (inputs NTT'd by the persistent batched
// transform k_ntt32_b, twiddles staged in shared memory) and the batched
// inverse transform, in place.  (A CTA per (prime, part, row) doing its own
// transforms with L2-resident twiddles ran at a third of that rate.)
__global__ void k_pointwise_mont(uint32_t* __restrict__ data, const uint32_t* __restrict__ m_ntt,
                                 int64_t stacks, int nparts, int k, int log_n, int m_broadcast,
                                 const Prime32Info* __restrict__ info) {
  // data: (B, nparts, k, N) NTT values; m_ntt: (B or 1, k, N) Montgomery form
  const int64_t n4 = (1ll << log_n) >> 2;
  const int64_t total = stacks * k * n4;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = g / n4, q = g - row * n4;  // row = (b * nparts + part) * k + j
    const int j = (int)(row % k);
    const int64_t b = row / ((int64_t)k * nparts);
    const Prime32Info inf = info[j];
    uint4* d = reinterpret_cast<uint4*>(data) + g;
    const uint4 m = reinterpret_cast<const uint4*>(m_ntt)[((m_broadcast ? 0 : b) * k + j) * n4 + q];
    uint4 v = *d;
    v.x = mulmod_mont_canon(v.x, m.x, inf);
    v.y = mulmod_mont_canon(v.y, m.y, inf);
    v.z = mulmod_mont_canon(v.z, m.z, inf);
    v.w = mulmod_mont_canon(v.w, m.w, inf);
    *d = v;
  }
}

__global__ void k_rows_mac_ntt(const uint32_t* __restrict__ x_ntt, const uint32_t* __restrict__ m_ntt,
                               const int32_t* __restrict__ row_ptr,
                               const int32_t* __restrict__ plain_seg,
                               const int32_t* __restrict__ plain_idx, uint32_t* __restrict__ out,
                               int64_t R, int k, int log_n, const Prime32Info* __restrict__ info) {
  // out (R, 2, k, N): row r, part, prime j, word i = sum over the row's
  // plaintexts p of x_ntt[seg p][part][j][i] * m_ntt[p][j][i] (x Montgomery)
  const int64_t n4 = (1ll << log_n) >> 2;
  const int64_t total = R * k * n4;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rj = g / n4, q = g - rj * n4;
    const int64_t r = rj / k;
    const int j = (int)(rj - r * k);
    const Prime32Info inf = info[j];
    const Mod32 md = make_mod(inf);
    uint32_t a0[4] = {0u, 0u, 0u, 0u}, a1[4] = {0u, 0u, 0u, 0u};
    for (int p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
      const int64_t seg = plain_seg[p];
      const int64_t mi = plain_idx != nullptr ? plain_idx[p] : p;
      const uint4 m = reinterpret_cast<const uint4*>(m_ntt)[(mi * k + j) * n4 + q];
      const uint4 x0 = reinterpret_cast<const uint4*>(x_ntt)[((seg * 2) * k + j) * n4 + q];
      const uint4 x1 = reinterpret_cast<const uint4*>(x_ntt)[((seg * 2 + 1) * k + j) * n4 + q];
      const uint32_t mv[4] = {m.x, m.y, m.z, m.w};
      const uint32_t xv0[4] = {x0.x, x0.y, x0.z, x0.w}, xv1[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        a0[e] = md.sub2p(a0[e] + mont_mul_lazy(mv[e], xv0[e], inf.p, inf.pinv_neg));
        a1[e] = md.sub2p(a1[e] + mont_mul_lazy(mv[e], xv1[e], inf.p, inf.pinv_neg));
      }
    }
    uint4* o = reinterpret_cast<uint4*>(out);
    o[((r * 2) * k + j) * n4 + q] = make_uint4(md.subp(a0[0]), md.subp(a0[1]), md.subp(a0[2]),
                                               md.subp(a0[3]));
    o[((r * 2 + 1) * k + j) * n4 + q] = make_uint4(md.subp(a1[0]), md.subp(a1[1]),
                                                   md.subp(a1[2]), md.subp(a1[3]));
  }
}

template <int LOGN>
static int run_mul_plain(hefv_ctx* c, const uint32_t* ct, const uint32_t* m, uint32_t* out,
                         int64_t B, int nparts, int bc, cudaStream_t st) {
  if (B <= 0) return 0;
  const int64_t stacks = B * nparts;
  if (int r = hefv_ntt_fwd32(c, ct, out, stacks, c->k, 0, 0, st)) return r;
  k_pointwise_mont<<<grid_for(stacks * c->k * ((int64_t)1 << LOGN) / 4, 256), 256, 0, st>>>(
      out, m, stacks, nparts, c->k, LOGN, bc, c->d_info32);
  HEFV_LAUNCH_CHECK("k_pointwise_mont");
  return hefv_ntt_inv32(c, out, out, stacks, c->k, 0, 0, st);
}

template <int LOGN>
static int run_rows_mac(hefv_ctx* c, const uint32_t* x, const uint32_t* m, const int32_t* rp,
                        const int32_t* seg, const int32_t* pidx, uint32_t* out, int64_t R,
                        cudaStream_t st) {
  if (R <= 0) return 0;
  k_rows_mac_ntt<<<grid_for(R * c->k * ((int64_t)1 << LOGN) / 4, 256), 256, 0, st>>>(
      x, m, rp, seg, pidx, out, R, c->k, LOGN, c->d_info32);
  HEFV_LAUNCH_CHECK("k_rows_mac_ntt");
  return hefv_ntt_inv32(c, out, out, 2 * R, c->k, 0, 0, st);
}

// ---------------------------------------------------------------------------
// Galois automorphism x -> x^g on coefficients (fv.py:157-173):
// out[m] = in[j1] if j1 = m g^-1 mod 2N < N, else -in[j1 - N].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512)
    k_automorph(const uint32_t* __restrict__ in, int64_t in_stride, const int32_t* __restrict__ slot,
                uint32_t* __restrict__ out, int nparts, int k, int log_n, uint32_t ginv,
                const Prime32Info* __restrict__ info) {
  extern __shared__ __align__(16) unsigned char smraw[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smraw);
  const int n = 1 << log_n;
  const int row = blockIdx.x;  // part * k + j
  const int j = row % k;
  const size_t b = blockIdx.y;
  const size_t src_ct = slot ? (size_t)slot[b] : b;
  const uint32_t* src = in + src_ct * in_stride + (size_t)row * n;
  uint32_t* dst = out + (b * nparts * k + row) * (size_t)n;
  const uint32_t p = info[j].p;
  // 16-byte coalesced staging of the source row
  for (int i = threadIdx.x; i < n / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = ld_stream_v4(reinterpret_cast<const uint4*>(src) + i);
  __syncthreads();
  const uint32_t mask = 2u * n - 1u;
  for (int q = threadIdx.x; q < n / 4; q += blockDim.x) {
    uint32_t v[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t m = 4u * q + r;
      const uint32_t j1 = (m * ginv) & mask;
      if (j1 < (uint32_t)n) {
        v[r] = sm[j1];
      } else {
        const uint32_t w = sm[j1 - n];
        v[r] = w ? p - w : 0u;
      }
    }
    reinterpret_cast<uint4*>(dst)[q] = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

// ---------------------------------------------------------------------------
// switch-key digit (fv.py:176-202) in the NTT domain
// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(Geo<LOGN, Loge32<LOGN>::v>::NT)
    k_keygen_digit(const uint32_t* __restrict__ a_i, const int8_t* __restrict__ e_i, int digit,
                   const uint32_t* __restrict__ gadget_i, const uint32_t* __restrict__ s_ntt,
                   const uint32_t* __restrict__ target_ntt, uint32_t* __restrict__ kbody,
                   uint32_t* __restrict__ kmask, int k, const uint2* __restrict__ tw_all,
                   const Prime32Info* __restrict__ info) {
  constexpr int LE = Loge32<LOGN>::v;
  typedef Geo<LOGN, LE> G_;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint32_t* sm = reinterpret_cast<uint32_t*>(smraw);
  const int j = blockIdx.x;
  const Prime32Info inf = info[j];
  const Mod32 md = make_mod(inf);
  const int tid = threadIdx.x;
  const size_t N = G_::N;
  uint32_t xa[G_::E], xe[G_::E];
#pragma unroll
  for (int e = 0; e < G_::E; ++e) {
    xa[e] = reduce_any(a_i[(size_t)j * N + tid + e * G_::NT], inf);
    xe[e] = small_to_mod(e_i[tid + e * G_::NT], inf.p);
  }
  cta_fwd<LOGN, LE, Mod32>(md, xa, sm, tw_all + (size_t)j * N);
  __syncthreads();
  cta_fwd<LOGN, LE, Mod32>(md, xe, sm, tw_all + (size_t)j * N);
  const uint32_t g = gadget_i[j];
  const size_t kofs = ((size_t)j * k + digit) * N;
  const uint32_t* sj = s_ntt + (size_t)j * N;
  const uint32_t* tj = target_ntt + (size_t)j * N;
#pragma unroll
  for (int e = 0; e < G_::E; ++e) {
    const uint32_t A = md.canon4(xa[e]);
    const uint32_t E = md.canon4(xe[e]);
    const uint32_t as_e = addmod(mulmod_small(A, sj[row_index<LOGN, LE>(tid, e)], inf), E, inf.p);
    const uint32_t gt = mulmod_small(g, tj[row_index<LOGN, LE>(tid, e)], inf);
    const uint32_t body = submod(gt, as_e, inf.p);
    kbody[kofs + row_index<LOGN, LE>(tid, e)] = mont_canon(body, inf);
    kmask[kofs + row_index<LOGN, LE>(tid, e)] = mont_canon(A, inf);
  }
}

template <int LOGN>
static int run_keygen_digit(hefv_ctx* c, const uint32_t* a_i, const int8_t* e_i, int digit,
                            const uint32_t* gad, const uint32_t* s, const uint32_t* tgt,
                            uint32_t* kb, uint32_t* km, cudaStream_t st) {
  typedef Geo<LOGN, Loge32<LOGN>::v> G_;
  auto kern = k_keygen_digit<LOGN>;
  if (int r = set_smem(kern, smem32<LOGN>())) return r;
  kern<<<c->k, G_::NT, smem32<LOGN>(), st>>>(a_i, e_i, digit, gad, s, tgt, kb, km, c->k,
                                             c->d_tw32, c->d_info32);
  HEFV_LAUNCH_CHECK("k_keygen_digit");
  return 0;
}

// ---------------------------------------------------------------------------
// layer output accumulation (inference.py:333-338) and batched bias adds
// ---------------------------------------------------------------------------
__global__ void k_accumulate_rows(const uint32_t* __restrict__ rows, const int32_t* __restrict__ seg,
                                  const int32_t* __restrict__ seg_out, uint32_t* __restrict__ out,
                                  int accumulate, int log_n, int k,
                                  const Prime32Info* __restrict__ info) {
  const int64_t ct_words = (int64_t)2 * k << log_n;
  const int m = blockIdx.y;
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= ct_words) return;
  const int j = (int)((w >> log_n) % k);
  const Prime32Info inf = info[j];
  uint64_t s = 0;
  const int lo = seg[m], hi = seg[m + 1];
  int cnt = 0;
  for (int r = lo; r < hi; ++r) {
    s += rows[(int64_t)r * ct_words + w];
    if (++cnt == 16) {  // keep s < 2^62 for the Barrett step
      s = barrett62(s, inf.p, inf.mu);
      cnt = 0;
    }
  }
  uint32_t v = barrett62(s, inf.p, inf.mu);
  uint32_t* o = out + (int64_t)seg_out[m] * ct_words + w;
  if (accumulate) v = addmod(v, *o, inf.p);
  *o = v;
}

__global__ void k_add_part0(uint32_t* __restrict__ rows, int64_t row_stride,
                            const int32_t* __restrict__ slot, const uint32_t* __restrict__ add,
                            int64_t P, int log_n, int k, const Prime32Info* __restrict__ info) {
  const int64_t stack = (int64_t)k << log_n;
  const int64_t total = P * stack;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pi = i / stack;
    const int64_t w = i - pi * stack;
    const int j = (int)(w >> log_n);
    uint32_t* o = rows + (int64_t)slot[pi] * row_stride + w;
    *o = addmod(*o, add[i], info[j].p);
  }
}

}  // namespace hefv

using namespace hefv;

extern "C" {

int hefv_encode(hefv_ctx* c, const uint64_t* slots, uint64_t* poly, int64_t B, void* stream) {
  if (int r = need_fv(c, "hefv_encode")) return r;
  HEFV_DISPATCH_FV(c->log_n, run_encode, c, slots, poly, B, as_stream(stream));
}

int hefv_decode(hefv_ctx* c, const uint64_t* poly, uint64_t* slots, int64_t B, void* stream) {
  if (int r = need_fv(c, "hefv_decode")) return r;
  HEFV_DISPATCH_FV(c->log_n, run_decode, c, poly, slots, B, as_stream(stream));
}

int hefv_encode_sparse(hefv_ctx* c, const int32_t* ptr, const int32_t* slot_idx,
                       const uint64_t* vals, uint64_t* poly, int64_t P, void* stream) {
  if (int r = need_fv(c, "hefv_encode_sparse")) return r;
  HEFV_DISPATCH_FV(c->log_n, run_encode_sparse, c, ptr, slot_idx, vals, poly, P,
                   as_stream(stream));
}

int hefv_plain_to_rns(hefv_ctx* c, const uint64_t* poly, uint32_t* out, int64_t B, int32_t mode,
                      int32_t to_ntt, int32_t montgomery, void* stream) {
  if (int r = need_fv(c, "hefv_plain_to_rns")) return r;
  if (mode != 0 && mode != 1) return fail("hefv_plain_to_rns: mode must be 0 or 1");
  HEFV_DISPATCH_FV(c->log_n, run_plain_to_rns, c, poly, out, B, mode, to_ntt, montgomery,
                   as_stream(stream));
}

int hefv_small_to_rns(hefv_ctx* c, const int8_t* small, uint32_t* out, int64_t B, int32_t to_ntt,
                      int32_t montgomery, void* stream) {
  if (int r = need_fv(c, "hefv_small_to_rns")) return r;
  HEFV_DISPATCH_FV(c->log_n, run_small_to_rns, c, small, out, B, to_ntt, montgomery,
                   as_stream(stream));
}

int hefv_elementwise(hefv_ctx* c, int32_t op, const uint32_t* a, const uint32_t* b,
                     const uint32_t* cc, uint32_t* out, int64_t rows, int64_t b_rows,
                     int64_t c_rows, void* stream) {
  if (int r = need_fv(c, "hefv_elementwise")) return r;
  if (op < 0 || op > 3) return fail("hefv_elementwise: bad op");
  if (rows <= 0) return 0;
  if (b_rows < 1 || (op == 3 && c_rows < 1)) return fail("hefv_elementwise: bad broadcast rows");
  const int64_t total = rows * ((int64_t)c->k << c->log_n);
  k_elementwise<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
      op, a, b, cc, out, total, c->log_n, c->k, b_rows, c_rows < 1 ? 1 : c_rows, c->d_info32);
  HEFV_LAUNCH_CHECK("k_elementwise");
  return 0;
}

int hefv_to_montgomery(hefv_ctx* c, const uint32_t* a, uint32_t* out, int64_t rows,
                       void* stream) {
  if (int r = need_fv(c, "hefv_to_montgomery")) return r;
  if (rows <= 0) return 0;
  const int64_t total = rows * ((int64_t)c->k << c->log_n);
  k_to_mont<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(a, out, total, c->log_n, c->k,
                                                                  c->d_info32);
  HEFV_LAUNCH_CHECK("k_to_mont");
  return 0;
}

int hefv_encrypt(hefv_ctx* c, const uint32_t* pk_ntt, const int8_t* u, const int8_t* e1,
                 const int8_t* e2, const uint32_t* dm, uint32_t* out, int64_t B, void* stream) {
  if (int r = need_fv(c, "hefv_encrypt")) return r;
  HEFV_DISPATCH_FV(c->log_n, run_encrypt, c, pk_ntt, u, e1, e2, dm, out, B, as_stream(stream));
}

int hefv_decrypt_round(hefv_ctx* c, const uint32_t* acc, uint64_t* out, int64_t B,
                       cudaStream_t st);  // mp_kernels.cu

int hefv_decrypt(hefv_ctx* c, const uint32_t* ct, int32_t nparts, const uint32_t* s_ntt,
                 const uint32_t* s2_ntt, uint64_t* out, uint32_t* scratch, int64_t B,
                 void* stream) {
  if (int r = need_fv(c, "hefv_decrypt")) return r;
  if (nparts < 2 || nparts > 3) return fail("hefv_decrypt: nparts must be 2 or 3");
  if (nparts == 3 && !s2_ntt) return fail("hefv_decrypt: 3-part ciphertext needs s^2");
  int r = 0;
  switch (c->log_n) {
#define HEFV_DC(L)                                                                          \
  case L:                                                                                   \
    r = run_decrypt_acc<L>(c, ct, nparts, s_ntt, s2_ntt, scratch, B, as_stream(stream));  \
    break;
    HEFV_DC(4)
    HEFV_DC(5)
    HEFV_DC(6)
    HEFV_DC(7)
    HEFV_DC(8)
    HEFV_DC(9)
    HEFV_DC(10)
    HEFV_DC(11)
    HEFV_DC(12)
    HEFV_DC(13)
    HEFV_DC(14)
#undef HEFV_DC
    default:
      return fail("hefv_decrypt: unsupported N");
  }
  if (r) return r;
  return hefv_decrypt_round(c, scratch, out, B, as_stream(stream));
}

int hefv_mul_plain(hefv_ctx* c, const uint32_t* ct, const uint32_t* m_ntt, uint32_t* out,
                   int64_t B, int32_t nparts, int32_t m_broadcast, void* stream) {
  if (int r = need_fv(c, "hefv_mul_plain")) return r;
  HEFV_DISPATCH_FV(c->log_n, run_mul_plain, c, ct, m_ntt, out, B, nparts, m_broadcast,
                   as_stream(stream));
}

int hefv_rows_mac(hefv_ctx* c, const uint32_t* x_ntt, const uint32_t* m_ntt,
                  const int32_t* row_ptr, const int32_t* plain_seg, uint32_t* out, int64_t R,
                  void* stream) {
  if (int r = need_fv(c, "hefv_rows_mac")) return r;
  HEFV_DISPATCH_FV(c->log_n, run_rows_mac, c, x_ntt, m_ntt, row_ptr, plain_seg,
                   (const int32_t*)nullptr, out, R, as_stream(stream));
}

int hefv_rows_mac_indexed(hefv_ctx* c, const uint32_t* x_ntt, const uint32_t* m_ntt,
                          const int32_t* row_ptr, const int32_t* tap_src,
                          const int32_t* tap_plain, uint32_t* out, int64_t R, void* stream) {
  if (int r = need_fv(c, "hefv_rows_mac_indexed")) return r;
  if (tap_plain == nullptr) return fail("hefv_rows_mac_indexed: tap_plain is NULL");
  HEFV_DISPATCH_FV(c->log_n, run_rows_mac, c, x_ntt, m_ntt, row_ptr, tap_src, tap_plain, out, R,
                   as_stream(stream));
}

int hefv_automorph(hefv_ctx* c, const uint32_t* in, int64_t in_stride, const int32_t* slot,
                   uint32_t* out, int32_t nparts, uint32_t galois_elt, int64_t B, void* stream) {
  if (int r = need_fv(c, "hefv_automorph")) return r;
  if (B <= 0) return 0;
  if (B > 65535) return fail("hefv_automorph: batch > 65535");
  if ((galois_elt & 1u) == 0) return fail("hefv_automorph: galois element must be odd");
  const uint32_t two_n = 2u * (uint32_t)c->n;
  // inverse of g mod 2N (2N is a power of two): Newton iteration
  uint32_t g = galois_elt % two_n, inv = 1;
  for (int it = 0; it < 6; ++it) inv *= 2u - g * inv;
  inv &= two_n - 1u;
  if (c->n < 16) return fail("hefv_automorph: N must be >= 16");
  const int threads = c->n / 4 >= 512 ? 512 : c->n / 4;
  const size_t smem = (size_t)c->n * 4;
  if (smem > 48 * 1024) {
    HEFV_CUDA(cudaFuncSetAttribute(k_automorph, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  }
  dim3 grid(nparts * c->k, (unsigned)B);
  k_automorph<<<grid, threads, smem, as_stream(stream)>>>(in, in_stride, slot, out, nparts, c->k,
                                                          c->log_n, inv, c->d_info32);
  HEFV_LAUNCH_CHECK("k_automorph");
  return 0;
}

int hefv_keygen_digit(hefv_ctx* c, const uint32_t* a_i, const int8_t* e_i, int32_t digit,
                      const uint32_t* gadget_i, const uint32_t* s_ntt,
                      const uint32_t* target_ntt, uint32_t* kbody, uint32_t* kmask,
                      void* stream) {
  if (int r = need_fv(c, "hefv_keygen_digit")) return r;
  if (digit < 0 || digit >= c->k) return fail("hefv_keygen_digit: digit out of range");
  HEFV_DISPATCH_FV(c->log_n, run_keygen_digit, c, a_i, e_i, digit, gadget_i, s_ntt, target_ntt,
                   kbody, kmask, as_stream(stream));
}

int hefv_accumulate_rows(hefv_ctx* c, const uint32_t* rows, const int32_t* seg,
                         const int32_t* seg_out, uint32_t* out, int32_t M, int32_t accumulate,
                         void* stream) {
  if (int r = need_fv(c, "hefv_accumulate_rows")) return r;
  if (M <= 0) return 0;
  if (M > 65535) return fail("hefv_accumulate_rows: too many segments");
  const int64_t ct_words = (int64_t)2 * c->k << c->log_n;
  dim3 grid((unsigned)((ct_words + 255) / 256), (unsigned)M);
  k_accumulate_rows<<<grid, 256, 0, as_stream(stream)>>>(rows, seg, seg_out, out, accumulate,
                                                         c->log_n, c->k, c->d_info32);
  HEFV_LAUNCH_CHECK("k_accumulate_rows");
  return 0;
}

int hefv_add_part0(hefv_ctx* c, uint32_t* rows, int64_t row_stride, const int32_t* slot,
                   const uint32_t* add, int64_t P, void* stream) {
  if (int r = need_fv(c, "hefv_add_part0")) return r;
  if (P <= 0) return 0;
  const int64_t total = P * ((int64_t)c->k << c->log_n);
  k_add_part0<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(rows, row_stride, slot, add, P,
                                                                    c->log_n, c->k, c->d_info32);
  HEFV_LAUNCH_CHECK("k_add_part0");
  return 0;
}

}  // extern "C"
