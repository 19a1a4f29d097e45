// Context creation: per-prime NTT tables and FV constants, built natively.
//
// Replaces the table construction of NttPrime.__init__ (reference
// ntt.py:149-189: psi powers, stage twiddles, N^{-1}, Shoup constants) and
// the constant part of _FvContext.__init__ (fv.py:78-110).  The tables are
// laid out for the merged-psi transforms in ntt.cuh: entry i of the forward
// table is psi^bitrev(i) (with its Shoup companion), entry i of the inverse
// table psi^-bitrev(i).
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/hefv.h"
#include "internal.h"

namespace hefv {

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_err = msg; }
int fail(const std::string& msg) {
  g_err = msg;
  return -1;
}
int check_cuda(cudaError_t e, const char* where) {
  g_err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  return -2;
}

static cudaEvent_t timing_event(hefv_ctx* c, cudaStream_t st) {
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  cudaEventRecord(e, st);
  c->ks_events.push_back(e);
  return e;
}
void ks_begin(hefv_ctx* c, int64_t B, cudaStream_t st) {
  c->ks_calls += 1;
  c->ks_cts += B;
  if (c->ks_timing) timing_event(c, st);
}
void ks_end(hefv_ctx* c, cudaStream_t st) {
  if (c->ks_timing) timing_event(c, st);
}
static void drop_ks_events(hefv_ctx* c) {
  for (cudaEvent_t e : c->ks_events)
    if (e) cudaEventDestroy(e);
  c->ks_events.clear();
}

typedef unsigned __int128 u128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }
static uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod(r, b, m);
    b = mulmod(b, b, m);
    e >>= 1;
  }
  return r;
}
static uint32_t bitrev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

// psi^bitrev(i) tables for one prime
static void make_tables(uint64_t p, uint64_t psi, int log_n, std::vector<uint64_t>& fwd,
                        std::vector<uint64_t>& inv) {
  const int n = 1 << log_n;
  std::vector<uint64_t> pw(n), ipw(n);
  const uint64_t ipsi = powmod(psi, p - 2, p);
  uint64_t a = 1, b = 1;
  for (int e = 0; e < n; ++e) {
    pw[e] = a;
    ipw[e] = b;
    a = mulmod(a, psi, p);
    b = mulmod(b, ipsi, p);
  }
  fwd.resize(n);
  inv.resize(n);
  for (int i = 0; i < n; ++i) {
    fwd[i] = pw[bitrev((uint32_t)i, log_n)];
    inv[i] = ipw[bitrev((uint32_t)i, log_n)];
  }
}

static int validate_root(uint64_t p, uint64_t psi, int log_n, std::string& why) {
  const uint64_t two_n = 2ull << log_n;
  if ((p - 1) % two_n != 0) {
    why = "prime " + std::to_string(p) + " is not 1 mod 2N";
    return -1;
  }
  if (powmod(psi, two_n >> 1, p) != p - 1) {
    why = "psi is not a primitive 2N-th root of unity mod " + std::to_string(p);
    return -1;
  }
  return 0;
}

}  // namespace hefv

using namespace hefv;

extern "C" {

const char* hefv_last_error(void) { return g_err.c_str(); }
int hefv_abi_version(void) { return 1; }
uint64_t hefv_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int hefv_ctx_create(hefv_ctx** out, uint32_t log_n, int32_t n32, const uint32_t* primes32,
                    const uint32_t* psi32, int32_t n64, const uint64_t* primes64,
                    const uint64_t* psi64) {
  if (!out) return fail("hefv_ctx_create: null out pointer");
  *out = nullptr;
  if (log_n < 1 || log_n > 16) return fail("hefv_ctx_create: log_n must be in [1, 16]");
  if (n32 < 0 || n64 < 0 || n32 + n64 == 0) return fail("hefv_ctx_create: empty prime set");
  hefv_ctx* c = new hefv_ctx();
  c->log_n = (int)log_n;
  c->n = 1 << log_n;
  const int n = c->n;
  std::string why;
  // ---- 32-bit primes
  c->n32 = n32;
  std::vector<uint2> tw((size_t)n32 * n), itw((size_t)n32 * n);
  std::vector<uint32_t> twm((size_t)n32 * n), itwm((size_t)n32 * n);
  for (int i = 0; i < n32; ++i) {
    const uint64_t p = primes32[i];
    if (p >= (1ull << 30) || p < 3) {
      delete c;
      return fail("hefv_ctx_create: word-sized primes must be below 2^30");
    }
    if (validate_root(p, psi32[i], log_n, why)) {
      delete c;
      return fail("hefv_ctx_create: " + why);
    }
    c->primes32.push_back((uint32_t)p);
    std::vector<uint64_t> f, v;
    make_tables(p, psi32[i], log_n, f, v);
    for (int j = 0; j < n; ++j) {
      tw[(size_t)i * n + j] = make_uint2((uint32_t)f[j], (uint32_t)((f[j] << 32) / p));
      itw[(size_t)i * n + j] = make_uint2((uint32_t)v[j], (uint32_t)((v[j] << 32) / p));
      twm[(size_t)i * n + j] = (uint32_t)((f[j] << 32) % p);
      itwm[(size_t)i * n + j] = (uint32_t)((v[j] << 32) % p);
    }
    Prime32Info inf{};
    inf.p = (uint32_t)p;
    uint32_t pinv = 1;  // Newton: p * pinv == 1 mod 2^32
    for (int it = 0; it < 5; ++it) pinv *= 2u - (uint32_t)p * pinv;
    inf.pinv_neg = (uint32_t)(0u - pinv);
    inf.pinv = pinv;
    inf.r2 = (uint32_t)(((u128)1 << 64) % p);
    inf.mu = (uint64_t)(((u128)1 << 64) / p);
    const uint64_t ninv = powmod((uint64_t)n, p - 2, p);
    inf.ninv = make_uint2((uint32_t)ninv, (uint32_t)((ninv << 32) / p));
    const uint64_t wn = mulmod(v[1], ninv, p);
    inf.wn = make_uint2((uint32_t)wn, (uint32_t)((wn << 32) / p));
    c->info32.push_back(inf);
  }
  // ---- 64-bit primes
  c->n64 = n64;
  std::vector<ulonglong2> tw64((size_t)n64 * n), itw64((size_t)n64 * n);
  for (int i = 0; i < n64; ++i) {
    const uint64_t p = primes64[i];
    if (p >= (1ull << 62) || p < 3) {
      delete c;
      return fail("hefv_ctx_create: 64-bit primes must be below 2^62");
    }
    if (validate_root(p, psi64[i], log_n, why)) {
      delete c;
      return fail("hefv_ctx_create: " + why);
    }
    c->primes64.push_back(p);
    std::vector<uint64_t> f, v;
    make_tables(p, psi64[i], log_n, f, v);
    for (int j = 0; j < n; ++j) {
      ulonglong2 a, b;
      a.x = f[j];
      a.y = (uint64_t)(((u128)f[j] << 64) / p);
      b.x = v[j];
      b.y = (uint64_t)(((u128)v[j] << 64) / p);
      tw64[(size_t)i * n + j] = a;
      itw64[(size_t)i * n + j] = b;
    }
    Prime64Info inf{};
    inf.p = p;
    const uint64_t ninv = powmod((uint64_t)n, p - 2, p);
    inf.ninv.x = ninv;
    inf.ninv.y = (uint64_t)(((u128)ninv << 64) / p);
    const uint64_t wn = mulmod(v[1], ninv, p);
    inf.wn.x = wn;
    inf.wn.y = (uint64_t)(((u128)wn << 64) / p);
    uint64_t pinv = 1;  // Newton: p * pinv == 1 mod 2^64
    for (int it = 0; it < 6; ++it) pinv *= 2ull - p * pinv;
    inf.pinv_neg = 0ull - pinv;
    {
      const u128 r = ((u128)1 << 64) % p;  // 2^64 mod p
      inf.r2 = (uint64_t)(r * r % p);
    }
    inf.mu = (uint64_t)(((u128)1 << 64) / p);
    c->info64.push_back(inf);
  }
  // ---- stream-ordered temporaries of the object-level ops (api.cu) come from
  // the device's default pool: keep freed blocks cached instead of returning
  // them to the driver at every synchronisation (a rotation hop would
  // otherwise map and unmap its key-switch scratch each call)
  {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 4ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  // ---- upload
  cudaError_t e = cudaSuccess;
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (e != cudaSuccess || bytes == 0) return;
    e = cudaMalloc(dst, bytes);
    if (e == cudaSuccess) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  up((void**)&c->d_tw32, tw.data(), tw.size() * sizeof(uint2));
  up((void**)&c->d_itw32, itw.data(), itw.size() * sizeof(uint2));
  up((void**)&c->d_info32, c->info32.data(), c->info32.size() * sizeof(Prime32Info));
  up((void**)&c->d_twm32, twm.data(), twm.size() * sizeof(uint32_t));
  up((void**)&c->d_itwm32, itwm.data(), itwm.size() * sizeof(uint32_t));
  up((void**)&c->d_tw64, tw64.data(), tw64.size() * sizeof(ulonglong2));
  up((void**)&c->d_itw64, itw64.data(), itw64.size() * sizeof(ulonglong2));
  up((void**)&c->d_info64, c->info64.data(), c->info64.size() * sizeof(Prime64Info));
  if (e != cudaSuccess) {
    hefv_ctx_destroy(c);
    return check_cuda(e, "hefv_ctx_create upload");
  }
  *out = c;
  return 0;
}

void hefv_ctx_destroy(hefv_ctx* c) {
  if (!c) return;
  cudaFree(c->d_tw32);
  cudaFree(c->d_itw32);
  cudaFree(c->d_info32);
  cudaFree(c->d_twm32);
  cudaFree(c->d_itwm32);
  cudaFree(c->d_tw64);
  cudaFree(c->d_itw64);
  cudaFree(c->d_info64);
  cudaFree(c->d_slot_to_dev);
  cudaFree(c->d_dev_to_slot);
  cudaFree(c->d_mp);
  cudaFree(c->d_delta);
  cudaFree(c->d_tmod);
  cudaFree(c->d_ksa_j);
  cudaFree(c->d_ks64a_t);
  cudaFree(c->d_ks64a_j);
  drop_ks_events(c);
  for (auto& sg : c->stages) {
    if (sg.done) {
      cudaEventSynchronize(sg.done);
      cudaEventDestroy(sg.done);
    }
    if (sg.host) cudaFreeHost(sg.host);
  }
  delete c;
}

int hefv_ks_timing(hefv_ctx* c, int32_t enable) {
  if (!c) return fail("hefv_ks_timing: null context");
  drop_ks_events(c);
  c->ks_calls = c->ks_cts = 0;
  c->ks_timing = enable != 0;
  return 0;
}

int hefv_ks_stats(hefv_ctx* c, int64_t* calls, int64_t* cts, double* ms) {
  if (!c) return fail("hefv_ks_stats: null context");
  if (calls) *calls = c->ks_calls;
  if (cts) *cts = c->ks_cts;
  if (ms) {
    double total = 0.0;
    for (size_t i = 0; i + 1 < c->ks_events.size(); i += 2) {
      HEFV_CUDA(cudaEventSynchronize(c->ks_events[i + 1]));
      float t = 0.f;
      HEFV_CUDA(cudaEventElapsedTime(&t, c->ks_events[i], c->ks_events[i + 1]));
      total += t;
    }
    *ms = total;
  }
  return 0;
}

int hefv_fv_setup(hefv_ctx* c, int32_t k, int32_t a, int32_t t_index, const int32_t* slot_to_ev,
                  int32_t wq, const uint32_t* q_words, const uint32_t* qhalf_words,
                  const uint32_t* qhat_words, const uint32_t* qhat_inv, int32_t wm,
                  const uint32_t* m_words, const uint32_t* mhalf_words,
                  const uint32_t* mhat_words, const uint32_t* mhat_inv,
                  const uint32_t* delta_mod) {
  if (!c) return fail("hefv_fv_setup: null context");
  if (k < 1 || a < 0 || k + a > c->n32) return fail("hefv_fv_setup: prime counts exceed context");
  if (t_index < 0 || t_index >= c->n64) return fail("hefv_fv_setup: bad t_index");
  // the exact t/q roundings divide by q with Knuth's algorithm D, which needs a
  // normalised divisor of at least two words (q >= 2^32: two or more q primes,
  // as FvParams.from_backend always chooses)
  if (wq < 2 || wq > 32) return fail("hefv_fv_setup: q must have 2..32 32-bit words (q >= 2^32)");
  if (wm > 64) return fail("hefv_fv_setup: aux product must have <= 64 words");
  for (int j = 0; j < k + a; ++j) {
    if (c->primes32[j] <= (1u << 28))
      return fail("hefv_fv_setup: FV primes must exceed 2^28 (lazy key-switch digits)");
  }
  const int n = c->n;
  c->k = k;
  c->a = a;
  c->t_index = t_index;
  c->t = c->primes64[t_index];
  c->wq = wq;
  c->wm = wm;
  // slot maps in device NTT order
  std::vector<int32_t> s2d(n / 2), d2s(n, -1);
  for (int s = 0; s < n / 2; ++s) {
    const int ev = slot_to_ev[s];
    if (ev < 0 || ev >= n) return fail("hefv_fv_setup: slot_to_ev out of range");
    const int dev = (int)bitrev((uint32_t)ev, c->log_n);
    s2d[s] = dev;
    d2s[dev] = s;
  }
  // multiprecision arena
  std::vector<uint32_t> mp;
  auto put = [&](const uint32_t* src, size_t cnt) {
    size_t off = mp.size();
    mp.insert(mp.end(), src, src + cnt);
    return off;
  };
  c->off_q = put(q_words, wq);
  c->off_qhalf = put(qhalf_words, wq);
  c->off_qhat = put(qhat_words, (size_t)k * wq);
  c->off_qhatinv = put(qhat_inv, k);
  // normalised q for long division (top bit of top word set)
  {
    int top = wq - 1;
    while (top > 0 && q_words[top] == 0) --top;
    if (top != wq - 1) return fail("hefv_fv_setup: q_words must not have a zero top word");
    uint32_t hw = q_words[wq - 1];
    int s = 0;
    while (!(hw & 0x80000000u)) {
      hw <<= 1;
      ++s;
    }
    c->q_shift = s;
    std::vector<uint32_t> qn(wq);
    for (int i = wq - 1; i >= 0; --i) {
      uint64_t v = (uint64_t)q_words[i] << s;
      if (s && i > 0) v |= (uint64_t)q_words[i - 1] >> (32 - s);
      qn[i] = (uint32_t)v;
    }
    c->off_qnorm = put(qn.data(), wq);
  }
  if (wm > 0) {
    c->off_m = put(m_words, wm);
    c->off_mhalf = put(mhalf_words, wm);
    c->off_mhat = put(mhat_words, (size_t)a * wm);
    c->off_mhatinv = put(mhat_inv, a);
  }
  std::vector<uint32_t> tmod(k);
  for (int j = 0; j < k; ++j) tmod[j] = (uint32_t)(c->t % c->primes32[j]);
  cudaFree(c->d_slot_to_dev);
  cudaFree(c->d_dev_to_slot);
  cudaFree(c->d_mp);
  cudaFree(c->d_delta);
  cudaFree(c->d_tmod);
  c->d_slot_to_dev = c->d_dev_to_slot = nullptr;
  c->d_mp = c->d_delta = c->d_tmod = nullptr;
  HEFV_CUDA(cudaMalloc(&c->d_slot_to_dev, s2d.size() * sizeof(int32_t)));
  HEFV_CUDA(cudaMemcpy(c->d_slot_to_dev, s2d.data(), s2d.size() * 4, cudaMemcpyHostToDevice));
  HEFV_CUDA(cudaMalloc(&c->d_dev_to_slot, d2s.size() * sizeof(int32_t)));
  HEFV_CUDA(cudaMemcpy(c->d_dev_to_slot, d2s.data(), d2s.size() * 4, cudaMemcpyHostToDevice));
  HEFV_CUDA(cudaMalloc(&c->d_mp, mp.size() * sizeof(uint32_t)));
  HEFV_CUDA(cudaMemcpy(c->d_mp, mp.data(), mp.size() * 4, cudaMemcpyHostToDevice));
  HEFV_CUDA(cudaMalloc(&c->d_delta, k * sizeof(uint32_t)));
  HEFV_CUDA(cudaMemcpy(c->d_delta, delta_mod, k * 4, cudaMemcpyHostToDevice));
  HEFV_CUDA(cudaMalloc(&c->d_tmod, k * sizeof(uint32_t)));
  HEFV_CUDA(cudaMemcpy(c->d_tmod, tmod.data(), k * 4, cudaMemcpyHostToDevice));
  c->fv_ready = true;
  return 0;
}

}  // extern "C"
