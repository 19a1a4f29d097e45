// 64-bit RNS key switch through an auxiliary basis of T ~29.4-bit NTT primes
// (config 4).  Same function as hefv_keyswitch64 / _keyswitch_apply
// (reference fv.py:205-217, object-dtype path for 50-62-bit primes):
//     d_j = iNTT_j( sum_i NTT_j(c_i mod p_j) * K_ji )  mod p_j
//         = ( sum_i c_i (*) B_ji ) mod p_j,    B_ji = iNTT_j(K_ji) in [0, p_j),
// with (*) the negacyclic product.  0 <= sum_i c_i (*) B_ji < k N max(p)^2,
// so it is computed EXACTLY in the aux basis a_0..a_{T-1} (A = prod a_t > 8 k
// N max(p)^2, checked by hefv_ks64_aux_setup) and reduced mod p_j -- the same
// canonical residues as the 64-bit path, with
//     T k   30-bit forward NTTs  instead of k^2 64-bit ones,
//     2 T k 30-bit inverse NTTs  instead of 2k 64-bit ones
// (a 64-bit butterfly costs ~4.5 30-bit ones on the integer pipes).
//
//   1. X[b][i][t]  = NTT_{a_t}(c_i mod a_t)          hefv_ntt32_fwd_rows64
//   2. Y[b][jp][t] = sum_i X[b][i][t] Ka[t][jp][i] mod a_t        k_ks64a_mac
//   3. y           = iNTT_{a_t}(Y)                   hefv_ntt_inv32 (batched)
//   4. out[b][jp]  = CRT_t(y (A/a_t)^-1) mod p_j                  k_ks64a_crt
//      v = round(sum_t y'_t / a_t) (fixed point; S / A < 1/8 keeps the
//      fraction within 1/8 of an integer), d = sum_t y'_t (A/a_t) - v A.
// Ka[t][part*k + j][i] = NTT_{a_t}(B_ji mod a_t) is built once per key by
// hefv_ks64_aux_key (jp = part * k + j; part 0 body, 1 mask).
#include <cmath>
#include <vector>

#include "../../include/hefv.h"
#include "internal.h"
#include "kcommon.cuh"

int hefv_ntt32_fwd_rows64(hefv_ctx* c, const uint64_t* in, uint32_t* out, int64_t rows,
                          int nprimes, int prime_base, cudaStream_t st);

namespace hefv {

constexpr int KS64A_TMAX = 6;
constexpr int KS64A_KMAX = 8;
constexpr int KS64A_CB = 16;  // ciphertexts per MAC CTA (key registers reused)
#ifndef KS64A_JG_V
#define KS64A_JG_V 2
#endif
constexpr int KS64A_JG = KS64A_JG_V;  // output rows per MAC thread

struct Ks64aT {  // per aux prime
  uint32_t a, pad;
  uint2 inv;      // (A / a_t)^-1 mod a_t, Shoup pair
  uint64_t mu;    // floor(2^64 / a_t) (Barrett)
  uint64_t r60;   // floor(2^60 / a_t) (quotient estimate)
};
struct Ks64aJ {  // per target prime
  ulonglong2 c[KS64A_TMAX];     // (A / a_t) mod p_j, Shoup pair
  uint64_t va[KS64A_TMAX + 1];  // (v A) mod p_j, v = 0..T
};

// Y[b][jp][t][n] = sum_i X[b][i][t][n] * Ka[t][jp][i][n] mod a_t for JG
// consecutive output rows jp = jg*JG .. of the 2k.  Thread = point n; CTA =
// (point block, t + T jg, ciphertext chunk); the JG x k key words of the point
// stay in registers and the next ciphertext's k digit words are loaded while
// the current one's products run.  sum < k a^2 < 2^62 (a < 2^29.5, k <= 8):
// one Barrett reduction.  (Staging the digit words in shared memory for all
// row groups of a point was measured 1.8x slower.)
template <int K, int JG>
__global__ void __launch_bounds__(128, JG <= 2 ? 6 : 4)
    k_ks64a_mac(const uint32_t* __restrict__ X, const uint32_t* __restrict__ ka,
                uint32_t* __restrict__ Y, int64_t B, int k, int T, int log_n,
                const Ks64aT* __restrict__ tc) {
  const int n = 1 << log_n;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % T, jg = blockIdx.y / T;
  if (w >= n) return;
  const Ks64aT c = tc[t];
  const int jp0 = jg * JG;
  const int nj = min(JG, 2 * k - jp0);
  uint32_t key[JG][K];
#pragma unroll
  for (int j = 0; j < JG; ++j)
#pragma unroll
    for (int i = 0; i < K; ++i)
      key[j][i] = (j < nj && i < k)
                      ? __ldg(ka + ((((size_t)t * 2 * k + jp0 + j) * k + i) << log_n) + w)
                      : 0u;
  const int64_t b0 = (int64_t)blockIdx.z * KS64A_CB;
  const int64_t b1 = min(B, b0 + KS64A_CB);
  const size_t xs = (size_t)T << log_n;  // digit stride in X, row stride in Y
  const uint32_t* xp = X + (((size_t)b0 * k * T + t) << log_n) + w;
  uint32_t* yp = Y + ((((size_t)b0 * 2 * k + jp0) * T + t) << log_n) + w;
  uint32_t x[K], xn[K];
#pragma unroll
  for (int i = 0; i < K; ++i) x[i] = (i < k && b0 < b1) ? __ldg(xp + i * xs) : 0u;
  for (int64_t b = b0; b < b1; ++b) {
    xp += (size_t)k * xs;
#pragma unroll
    for (int i = 0; i < K; ++i) xn[i] = (i < k && b + 1 < b1) ? __ldg(xp + i * xs) : 0u;
#pragma unroll
    for (int j = 0; j < JG; ++j) {
      if (j < nj) {
        uint64_t s = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) s += (uint64_t)x[i] * key[j][i];
        yp[j * xs] = barrett62(s, c.a, c.mu);
      }
    }
    yp += (size_t)2 * k * xs;
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = xn[i];
  }
}

// out[b][part][j][n] = CRT over t of y[b][part*k + j][t][n] reduced mod p_j.
// Thread = 4 consecutive points (16-byte loads of y, four independent
// accumulation chains); the per-prime constants sit in shared memory.
__global__ void __launch_bounds__(256)
    k_ks64a_crt(const uint32_t* __restrict__ y, uint64_t* __restrict__ out, int k, int T,
                int log_n, int64_t rows, const Ks64aT* __restrict__ tc,
                const Ks64aJ* __restrict__ jc, const Prime64Info* __restrict__ info) {
  __shared__ Ks64aT st[KS64A_TMAX];
  __shared__ Ks64aJ sj;
  const int n = 1 << log_n;
  const int row = blockIdx.y + blockIdx.z * 65535;  // b * 2k + jp (< 2^31)
  if (row >= rows) return;
  const int j = (row % (2 * k)) % k;
  if (threadIdx.x < T) st[threadIdx.x] = tc[threadIdx.x];
  if (threadIdx.x == 0) sj = jc[j];
  __syncthreads();
  const int w = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (w >= n) return;
  const uint64_t p = info[j].p, p2 = 2 * p;
  uint64_t frac[4] = {0, 0, 0, 0}, acc[4] = {0, 0, 0, 0};
  const uint32_t* yr = y + ((size_t)row * T << log_n) + w;
#pragma unroll
  for (int t = 0; t < KS64A_TMAX; ++t) {
    if (t < T) {
      const Ks64aT c = st[t];
      const ulonglong2 cc = sj.c[t];
      const uint4 v4 = *reinterpret_cast<const uint4*>(yr + ((size_t)t << log_n));
      const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t yt = Mod32::mul_shoup(vv[q], c.inv.x, c.inv.y, c.a);
        yt = yt >= c.a ? yt - c.a : yt;         // canonical y'_t
        frac[q] += (uint64_t)yt * c.r60;         // y'_t / a_t in 4.60 fixed point
        acc[q] += Mod64::mul_shoup(yt, cc.x, cc.y, p);  // [0, 2p) per term
        acc[q] = acc[q] >= p2 ? acc[q] - p2 : acc[q];
      }
    }
  }
  uint64_t r[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int v = (int)((frac[q] + (1ull << 59)) >> 60);
    uint64_t x = acc[q] + (p - sj.va[v]);  // < 3p
    x = x >= p2 ? x - p2 : x;
    r[q] = x >= p ? x - p : x;
  }
  ulonglong2* o = reinterpret_cast<ulonglong2*>(out + ((size_t)row << log_n) + w);
  o[0] = make_ulonglong2(r[0], r[1]);
  o[1] = make_ulonglong2(r[2], r[3]);
}

// key conversion helpers (setup only)
// in: (2, k_j, k_i, N) [part][j][i]  ->  out: (2, k_i, k_j, N) [part][i][j]
__global__ void k_ks64a_key_t(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int k,
                              int log_n) {
  const int n = 1 << log_n;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n) return;
  const int r = blockIdx.y;  // (part, j, i)
  const int i = r % k, j = (r / k) % k, part = r / (k * k);
  out[((((size_t)part * k + i) * k + j) << log_n) + w] = in[((size_t)r << log_n) + w];
}
// in: (2k_i k_j rows, T, N) [part][i][j][t]  ->  Ka: (T, 2k, k, N) [t][part k + j][i]
__global__ void k_ks64a_key_p(const uint32_t* __restrict__ in, uint32_t* __restrict__ ka, int k,
                              int T, int log_n) {
  const int n = 1 << log_n;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n) return;
  const int r = blockIdx.y;  // ((part, i, j), t)
  const int t = r % T, row = r / T;
  const int j = row % k, i = (row / k) % k, part = row / (k * k);
  ka[((((size_t)t * 2 * k + part * k + j) * k + i) << log_n) + w] = in[((size_t)r << log_n) + w];
}

}  // namespace hefv

using namespace hefv;

namespace {
using u128 = unsigned __int128;
uint64_t powmod64(uint64_t a, uint64_t e, uint64_t m) {
  u128 r = 1 % m, x = a % m;
  while (e) {
    if (e & 1) r = r * x % m;
    x = x * x % m;
    e >>= 1;
  }
  return (uint64_t)r;
}
}  // namespace

extern "C" {

int hefv_ks64_aux_setup(hefv_ctx* c, int32_t T) {
  if (!c) return fail("hefv_ks64_aux_setup: null context");
  const int k = c->n64;
  if (T < 2 || T > KS64A_TMAX || T != c->n32)
    return fail("hefv_ks64_aux_setup: the context's 32-bit primes must be the T aux primes");
  if (k < 1 || k > KS64A_KMAX) return fail("hefv_ks64_aux_setup: 1..8 64-bit primes");
  // exactness: A > 8 k N max(p)^2, and the MAC bound k a^2 < 2^62
  double logA = 0, logp = 0;
  for (int t = 0; t < T; ++t) {
    const double a = (double)c->primes32[t];
    if (a * a * k >= std::ldexp(1.0, 62)) return fail("hefv_ks64_aux_setup: aux prime too large");
    logA += std::log2(a);
  }
  for (int j = 0; j < k; ++j) logp = std::max(logp, std::log2((double)c->primes64[j]));
  if (logA < 3.0 + std::log2((double)k) + c->log_n + 2 * logp + 0.01)
    return fail("hefv_ks64_aux_setup: aux basis too small for exactness");
  // A mod a_t, A/a_t mod m via products
  std::vector<Ks64aT> tv(T);
  std::vector<Ks64aJ> jv(k);
  for (int t = 0; t < T; ++t) {
    const uint64_t a = c->primes32[t];
    uint64_t ahat = 1;  // (A / a_t) mod a_t
    for (int s = 0; s < T; ++s)
      if (s != t) ahat = (uint64_t)((u128)ahat * (c->primes32[s] % a) % a);
    const uint64_t inv = powmod64(ahat, a - 2, a);
    tv[t].a = (uint32_t)a;
    tv[t].inv = make_uint2((uint32_t)inv, (uint32_t)(((uint64_t)inv << 32) / a));
    tv[t].mu = (uint64_t)(((u128)1 << 64) / a);
    tv[t].r60 = (uint64_t)((1ull << 60) / a);
  }
  for (int j = 0; j < k; ++j) {
    const uint64_t p = c->primes64[j];
    uint64_t Amod = 1;
    for (int t = 0; t < T; ++t) Amod = (uint64_t)((u128)Amod * c->primes32[t] % p);
    for (int t = 0; t < T; ++t) {
      uint64_t ch = 1;
      for (int s = 0; s < T; ++s)
        if (s != t) ch = (uint64_t)((u128)ch * c->primes32[s] % p);
      jv[j].c[t] = make_ulonglong2(ch, (uint64_t)(((u128)ch << 64) / p));
    }
    for (int v = 0; v <= T; ++v) jv[j].va[v] = (uint64_t)((u128)Amod * v % p);
  }
  cudaFree(c->d_ks64a_t);
  cudaFree(c->d_ks64a_j);
  c->d_ks64a_t = nullptr;
  c->d_ks64a_j = nullptr;
  HEFV_CUDA(cudaMalloc(&c->d_ks64a_t, T * sizeof(Ks64aT)));
  HEFV_CUDA(cudaMalloc(&c->d_ks64a_j, k * sizeof(Ks64aJ)));
  HEFV_CUDA(cudaMemcpy(c->d_ks64a_t, tv.data(), T * sizeof(Ks64aT), cudaMemcpyHostToDevice));
  HEFV_CUDA(cudaMemcpy(c->d_ks64a_j, jv.data(), k * sizeof(Ks64aJ), cudaMemcpyHostToDevice));
  c->ks64a_T = T;
  return 0;
}

int hefv_keyswitch64_aux(hefv_ctx* c, const uint32_t* kaux, const uint64_t* digits,
                         uint64_t* out, uint32_t* scratch, int64_t B, void* stream) {
  if (!c || c->ks64a_T == 0) return fail("hefv_keyswitch64_aux: run hefv_ks64_aux_setup first");
  if (B <= 0) return 0;
  const int k = c->n64, T = c->ks64a_T;
  const int64_t n = c->n;
  cudaStream_t st = as_stream(stream);
  uint32_t* X = scratch;                       // (B, k, T, N)
  uint32_t* Y = scratch + (size_t)B * k * T * n;  // (B, 2k, T, N)
  if (int r = hefv_ntt32_fwd_rows64(c, digits, X, B * k, T, 0, st)) return r;
  {
    constexpr int JG = KS64A_JG;
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)(T * ((2 * k + JG - 1) / JG)),
              (unsigned)((B + KS64A_CB - 1) / KS64A_CB));
    if (grid.z > 65535) return fail("hefv_keyswitch64_aux: batch too large");
    const Ks64aT* tcp = reinterpret_cast<const Ks64aT*>(c->d_ks64a_t);
    if (k <= 4)
      k_ks64a_mac<4, JG><<<grid, 128, 0, st>>>(X, kaux, Y, B, k, T, c->log_n, tcp);
    else
      k_ks64a_mac<8, JG><<<grid, 128, 0, st>>>(X, kaux, Y, B, k, T, c->log_n, tcp);
    HEFV_LAUNCH_CHECK("k_ks64a_mac");
  }
  if (int r = hefv_ntt_inv32(c, Y, Y, B * 2 * k, T, 0, 0, stream)) return r;
  {
    const int64_t rows = B * 2 * k;
    if (rows > 0x7fffffff) return fail("hefv_keyswitch64_aux: batch too large");
    dim3 grid((unsigned)((n / 4 + 255) / 256), (unsigned)(rows < 65535 ? rows : 65535),
              (unsigned)((rows + 65534) / 65535));
    k_ks64a_crt<<<grid, 256, 0, st>>>(Y, out, k, T, c->log_n, rows,
                                      reinterpret_cast<const Ks64aT*>(c->d_ks64a_t),
                                      reinterpret_cast<const Ks64aJ*>(c->d_ks64a_j), c->d_info64);
    HEFV_LAUNCH_CHECK("k_ks64a_crt");
  }
  return 0;
}

// Aux-basis form of a switch key: kbody/kmask (k, k, N) = [target j][digit
// i], device NTT order, PLAIN residues (not Montgomery); kaux: (T, 2k, k, N)
// u32; scratch: >= (4 + T) k k N u64 words.
int hefv_ks64_aux_key(hefv_ctx* c, const uint64_t* kbody, const uint64_t* kmask, uint32_t* kaux,
                      uint64_t* scratch, void* stream) {
  if (!c || c->ks64a_T == 0) return fail("hefv_ks64_aux_key: run hefv_ks64_aux_setup first");
  const int k = c->n64, T = c->ks64a_T;
  const int64_t n = c->n, kk = (int64_t)k * k;
  cudaStream_t st = as_stream(stream);
  uint64_t* kin = scratch;              // (2, k, k, N) [part][j][i]
  uint64_t* kt = scratch + 2 * kk * n;  // (2, k, k, N) [part][i][j]
  uint32_t* rows = reinterpret_cast<uint32_t*>(scratch + 4 * kk * n);  // (2 k k, T, N) u32
  HEFV_CUDA(cudaMemcpyAsync(kin, kbody, kk * n * 8, cudaMemcpyDeviceToDevice, st));
  HEFV_CUDA(cudaMemcpyAsync(kin + kk * n, kmask, kk * n * 8, cudaMemcpyDeviceToDevice, st));
  dim3 g1((unsigned)((n + 255) / 256), (unsigned)(2 * kk));
  k_ks64a_key_t<<<g1, 256, 0, st>>>(kin, kt, k, c->log_n);
  HEFV_LAUNCH_CHECK("k_ks64a_key_t");
  // B_ji = iNTT_j(K_ji): rows (part, i) x prime j
  if (int r = hefv_ntt_inv64(c, kt, kt, 2 * k, k, 0, 0, stream)) return r;
  if (int r = hefv_ntt32_fwd_rows64(c, kt, rows, 2 * kk, T, 0, st)) return r;
  dim3 g2((unsigned)((n + 255) / 256), (unsigned)(2 * kk * T));
  k_ks64a_key_p<<<g2, 256, 0, st>>>(rows, kaux, k, T, c->log_n);
  HEFV_LAUNCH_CHECK("k_ks64a_key_p");
  return 0;
}

}  // extern "C"
