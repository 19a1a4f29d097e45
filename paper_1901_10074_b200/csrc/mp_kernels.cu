// Exact multiprecision kernels: the two big-integer roundings of BFV.
//
//   * decryption rounding m = floor((x t + floor(q/2)) / q) mod t with
//     x = CRT_q(acc) in [0, q)                     -- reference fv.py:348-349
//   * the ct x ct tensor (K8): centred CRT lift q -> auxiliary basis,
//     NTT-domain tensor under every auxiliary prime, then per stack
//     x = centred CRT_M(stack), y = floor((x t + floor(q/2)) / q) mod q,
//     back to the q basis                          -- reference fv.py:377-409
//
// One thread per coefficient; numbers are little-endian 32-bit words in
// thread-local arrays.  CRT uses x = sum_i y_i * (P/p_i) - v * P with
// y_i = r_i (P/p_i)^-1 mod p_i and v = floor(sum_i y_i / p_i), v estimated in
// double precision from below and corrected by an exact comparison; the
// division by q is Knuth's algorithm D.  No approximate (BEHZ/HPS) rounding
// is used anywhere, so the result equals Python's big-integer arithmetic.
#include <algorithm>
#include <cmath>

#include "../../include/hefv.h"
#include "internal.h"
#include "kcommon.cuh"

namespace hefv {

constexpr int MAXWQ = 32;
constexpr int MAXWM = 64;

__device__ __forceinline__ uint32_t mulmod_sm(uint32_t a, uint32_t b, const Prime32Info& inf) {
  return barrett62((uint64_t)a * b, inf.p, inf.mu);
}

// x[0..W] = CRT reconstruction in [0, P) of residues res[i * rstride]
// under primes info[base + i], i < nres.
__device__ void mp_crt(const uint32_t* __restrict__ res, size_t rstride, int nres, int base,
                       const uint32_t* __restrict__ hat, const uint32_t* __restrict__ hatinv,
                       const uint32_t* __restrict__ modw, int W,
                       const Prime32Info* __restrict__ info, uint32_t* x) {
  for (int w = 0; w <= W; ++w) x[w] = 0;
  double f = 0.0;
  for (int i = 0; i < nres; ++i) {
    const Prime32Info inf = info[base + i];
    const uint32_t y = mulmod_sm(res[(size_t)i * rstride], hatinv[i], inf);
    f += (double)y / (double)inf.p;
    uint64_t carry = 0;
    const uint32_t* h = hat + (size_t)i * W;
    for (int w = 0; w < W; ++w) {
      const uint64_t t = (uint64_t)y * h[w] + x[w] + carry;
      x[w] = (uint32_t)t;
      carry = t >> 32;
    }
    x[W] += (uint32_t)carry;
  }
  // v_est <= v = floor(f_exact) and v_est >= v - 1
  double fe = f - 9.094947017729282e-13;  // 2^-40
  uint32_t v = fe > 0.0 ? (uint32_t)floor(fe) : 0u;
  if (v) {
    int64_t k = 0;
    for (int w = 0; w < W; ++w) {
      const uint64_t p = (uint64_t)v * modw[w];
      const int64_t t = (int64_t)x[w] - k - (int64_t)(p & 0xffffffffull);
      x[w] = (uint32_t)t;
      k = (int64_t)(p >> 32) - (t >> 32);
    }
    x[W] = (uint32_t)((int64_t)x[W] - k);
  }
  // at most one more subtraction of P
  bool ge = x[W] != 0;
  if (!ge) {
    ge = true;
    for (int w = W - 1; w >= 0; --w) {
      if (x[w] != modw[w]) {
        ge = x[w] > modw[w];
        break;
      }
    }
  }
  if (ge) {
    int64_t br = 0;
    for (int w = 0; w < W; ++w) {
      const int64_t t = (int64_t)x[w] - modw[w] - br;
      x[w] = (uint32_t)t;
      br = t < 0 ? 1 : 0;
    }
    x[W] -= (uint32_t)br;
  }
}

// compare a (W words) with b (W words): -1, 0, 1
__device__ __forceinline__ int mp_cmp(const uint32_t* a, const uint32_t* b, int W) {
  for (int w = W - 1; w >= 0; --w) {
    if (a[w] != b[w]) return a[w] > b[w] ? 1 : -1;
  }
  return 0;
}

// out = a - b (W words, a >= b)
__device__ __forceinline__ void mp_sub(const uint32_t* a, const uint32_t* b, uint32_t* out, int W) {
  int64_t br = 0;
  for (int w = 0; w < W; ++w) {
    const int64_t t = (int64_t)a[w] - b[w] - br;
    out[w] = (uint32_t)t;
    br = t < 0 ? 1 : 0;
  }
}

// z[0..W+1] = a[0..W-1] * t (t < 2^64)
__device__ __forceinline__ void mp_mul_u64(const uint32_t* a, int W, uint64_t t, uint32_t* z) {
  const uint32_t t0 = (uint32_t)t, t1 = (uint32_t)(t >> 32);
  for (int w = 0; w < W + 2; ++w) z[w] = 0;
  uint64_t c = 0;
  for (int w = 0; w < W; ++w) {
    const uint64_t s = (uint64_t)a[w] * t0 + z[w] + c;
    z[w] = (uint32_t)s;
    c = s >> 32;
  }
  z[W] = (uint32_t)c;
  c = 0;
  for (int w = 0; w < W; ++w) {
    const uint64_t s = (uint64_t)a[w] * t1 + z[w + 1] + c;
    z[w + 1] = (uint32_t)s;
    c = s >> 32;
  }
  z[W + 1] = (uint32_t)c;
}

// z[0..nz-1] += b[0..nb-1] (nz >= nb), carry dropped past nz
__device__ __forceinline__ void mp_add_into(uint32_t* z, int nz, const uint32_t* b, int nb) {
  uint64_t c = 0;
  for (int w = 0; w < nz; ++w) {
    const uint64_t s = (uint64_t)z[w] + (w < nb ? b[w] : 0u) + c;
    z[w] = (uint32_t)s;
    c = s >> 32;
  }
}

// z -= b (z >= b)
__device__ __forceinline__ void mp_sub_into(uint32_t* z, int nz, const uint32_t* b, int nb) {
  int64_t br = 0;
  for (int w = 0; w < nz; ++w) {
    const int64_t t = (int64_t)z[w] - (w < nb ? b[w] : 0u) - br;
    z[w] = (uint32_t)t;
    br = t < 0 ? 1 : 0;
  }
}

// Knuth D: quotient of u (nu words) by the divisor whose normalised form is
// vn (W words, top bit set, normalisation shift s).  un: scratch of nu + 1
// words; qw receives nu - W + 1 words.  Requires nu >= W >= 2.
__device__ void mp_div(const uint32_t* u, int nu, const uint32_t* __restrict__ vn, int W, int s,
                       uint32_t* un, uint32_t* qw) {
  un[nu] = s ? (u[nu - 1] >> (32 - s)) : 0u;
  for (int i = nu - 1; i > 0; --i) un[i] = s ? ((u[i] << s) | (u[i - 1] >> (32 - s))) : u[i];
  un[0] = u[0] << s;
  const uint64_t b = 1ull << 32;
  const uint64_t vtop = vn[W - 1], vnext = vn[W - 2];
  for (int j = nu - W; j >= 0; --j) {
    const uint64_t num = ((uint64_t)un[j + W] << 32) | un[j + W - 1];
    uint64_t qhat = num / vtop;
    uint64_t rhat = num - qhat * vtop;
    while (qhat >= b || qhat * vnext > ((rhat << 32) | un[j + W - 2])) {
      --qhat;
      rhat += vtop;
      if (rhat >= b) break;
    }
    int64_t k = 0, t;
    for (int i = 0; i < W; ++i) {
      const uint64_t p = qhat * vn[i];
      t = (int64_t)un[i + j] - k - (int64_t)(p & 0xffffffffull);
      un[i + j] = (uint32_t)t;
      k = (int64_t)(p >> 32) - (t >> 32);
    }
    t = (int64_t)un[j + W] - k;
    un[j + W] = (uint32_t)t;
    if (t < 0) {
      --qhat;
      uint64_t c = 0;
      for (int i = 0; i < W; ++i) {
        const uint64_t sum = (uint64_t)un[i + j] + vn[i] + c;
        un[i + j] = (uint32_t)sum;
        c = sum >> 32;
      }
      un[j + W] += (uint32_t)c;
    }
    qw[j] = (uint32_t)qhat;
  }
}

// x (W words) mod p via Horner with Barrett steps
__device__ __forceinline__ uint32_t mp_mod_small(const uint32_t* x, int W, const Prime32Info& inf) {
  uint32_t r = 0;
  for (int w = W - 1; w >= 0; --w) r = barrett62(((uint64_t)r << 32) | x[w], inf.p, inf.mu);
  return r;
}

struct MpConsts {
  const uint32_t* q;
  const uint32_t* qhalf;
  const uint32_t* qhat;
  const uint32_t* qhatinv;
  const uint32_t* qnorm;
  const uint32_t* m;
  const uint32_t* mhalf;
  const uint32_t* mhat;
  const uint32_t* mhatinv;
  int wq, wm, qshift, k, a, log_n;
  uint64_t t;
};

static MpConsts mp_consts(const hefv_ctx* c) {
  MpConsts m;
  m.q = c->d_mp + c->off_q;
  m.qhalf = c->d_mp + c->off_qhalf;
  m.qhat = c->d_mp + c->off_qhat;
  m.qhatinv = c->d_mp + c->off_qhatinv;
  m.qnorm = c->d_mp + c->off_qnorm;
  m.m = c->d_mp + c->off_m;
  m.mhalf = c->d_mp + c->off_mhalf;
  m.mhat = c->d_mp + c->off_mhat;
  m.mhatinv = c->d_mp + c->off_mhatinv;
  m.wq = c->wq;
  m.wm = c->wm;
  m.qshift = c->q_shift;
  m.k = c->k;
  m.a = c->a;
  m.log_n = c->log_n;
  m.t = c->t;
  return m;
}

// ---- decryption rounding -------------------------------------------------
__global__ void __launch_bounds__(128)
    k_decrypt_round(const uint32_t* __restrict__ acc, uint64_t* __restrict__ out, int64_t B,
                    MpConsts mc, const Prime32Info* __restrict__ info) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = 1ll << mc.log_n;
  if (gid >= B * n) return;
  const int64_t b = gid >> mc.log_n;
  const int64_t i = gid & (n - 1);
  uint32_t x[MAXWQ + 1], z[MAXWQ + 3], un[MAXWQ + 4], qw[4];
  mp_crt(acc + b * mc.k * n + i, (size_t)n, mc.k, 0, mc.qhat, mc.qhatinv, mc.q, mc.wq, info, x);
  mp_mul_u64(x, mc.wq, mc.t, z);           // z: wq + 2 words
  mp_add_into(z, mc.wq + 2, mc.qhalf, mc.wq);
  mp_div(z, mc.wq + 2, mc.qnorm, mc.wq, mc.qshift, un, qw);  // 3 quotient words
  uint64_t y = ((uint64_t)qw[1] << 32) | qw[0];
  if (y >= mc.t) y -= mc.t;
  out[gid] = y;
}

// ---- ct x ct: centred lift q -> aux --------------------------------------
// in: nparts ciphertext parts, each (k, N); out: (nparts, a, N)
__global__ void __launch_bounds__(128)
    k_mult_lift(const uint32_t* __restrict__ a, int64_t a_stride, const uint32_t* __restrict__ b,
                int64_t b_stride, int nparts, uint32_t* __restrict__ out, MpConsts mc,
                const Prime32Info* __restrict__ info) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = 1ll << mc.log_n;
  if (gid >= nparts * n) return;
  const int64_t ct = blockIdx.y;
  const int part = (int)(gid >> mc.log_n);
  const int64_t i = gid & (n - 1);
  const int64_t stack_q = (int64_t)mc.k * n;
  const uint32_t* src = part < 2 ? a + ct * a_stride + part * stack_q
                                 : b + ct * b_stride + (part - 2) * stack_q;
  out += ct * nparts * (int64_t)mc.a * n;
  uint32_t x[MAXWQ + 1], mag[MAXWQ];
  mp_crt(src + i, (size_t)n, mc.k, 0, mc.qhat, mc.qhatinv, mc.q, mc.wq, info, x);
  const bool neg = mp_cmp(x, mc.qhalf, mc.wq) > 0;  // x > floor(q/2) -> x - q
  if (neg)
    mp_sub(mc.q, x, mag, mc.wq);
  else
    for (int w = 0; w < mc.wq; ++w) mag[w] = x[w];
  uint32_t* dst = out + (int64_t)part * mc.a * n + i;
  for (int ai = 0; ai < mc.a; ++ai) {
    const Prime32Info inf = info[mc.k + ai];
    uint32_t r = mp_mod_small(mag, mc.wq, inf);
    if (neg && r) r = inf.p - r;
    dst[(int64_t)ai * n] = r;
  }
}

// ---- ct x ct: NTT-domain tensor under each aux prime ----------------------
// L: (4 or 2, a, N) device-order NTTs (a0, a1, b0, b1); T: (3, a, N)
__global__ void k_mult_tensor(const uint32_t* __restrict__ L, int same, uint32_t* __restrict__ T,
                              MpConsts mc, const Prime32Info* __restrict__ info) {
  const int64_t n = 1ll << mc.log_n;
  const int64_t stack = (int64_t)mc.a * n;
  L += (int64_t)blockIdx.y * (same ? 2 : 4) * stack;
  T += (int64_t)blockIdx.y * 3 * stack;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < stack;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int ai = (int)(g >> mc.log_n);
    const Prime32Info inf = info[mc.k + ai];
    const uint32_t a0 = L[g], a1 = L[stack + g];
    const uint32_t b0 = same ? a0 : L[2 * stack + g];
    const uint32_t b1 = same ? a1 : L[3 * stack + g];
    T[g] = mulmod_sm(a0, b0, inf);
    uint32_t s = mulmod_sm(a0, b1, inf) + mulmod_sm(a1, b0, inf);
    T[stack + g] = s >= inf.p ? s - inf.p : s;
    T[2 * stack + g] = mulmod_sm(a1, b1, inf);
  }
}

// ---- ct x ct: exact t/q scale-and-round back to the q basis ----------------
// T: (3, a, N) coefficient domain; out: (3, k, N)
__global__ void __launch_bounds__(64)
    k_mult_scale(const uint32_t* __restrict__ T, uint32_t* __restrict__ out, MpConsts mc,
                 const Prime32Info* __restrict__ info) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = 1ll << mc.log_n;
  if (gid >= 3 * n) return;
  T += (int64_t)blockIdx.y * 3 * mc.a * n;
  out += (int64_t)blockIdx.y * 3 * mc.k * n;
  const int st = (int)(gid >> mc.log_n);
  const int64_t i = gid & (n - 1);
  uint32_t x[MAXWM + 1], z[MAXWM + 3], un[MAXWM + 4], qw[MAXWM + 3];
  mp_crt(T + (int64_t)st * mc.a * n + i, (size_t)n, mc.a, mc.k, mc.mhat, mc.mhatinv, mc.m, mc.wm,
         info, x);
  const bool neg = mp_cmp(x, mc.mhalf, mc.wm) > 0;
  if (neg) mp_sub(mc.m, x, x, mc.wm);  // magnitude M - x
  // z = |x| * t  (wm + 2 words)
  const int nz = mc.wm + 2;
  mp_mul_u64(x, mc.wm, mc.t, z);
  bool yneg = false, yzero = false;
  if (!neg) {
    mp_add_into(z, nz, mc.qhalf, mc.wq);
  } else {
    // compare |x| t with floor(q/2)
    bool le = true;
    for (int w = nz - 1; w >= 0; --w) {
      const uint32_t hw = w < mc.wq ? mc.qhalf[w] : 0u;
      if (z[w] != hw) {
        le = z[w] < hw;
        break;
      }
    }
    if (le) {
      yzero = true;
    } else {
      // y = -ceil((|x| t - h) / q) = -floor((|x| t - h + q - 1) / q)
      mp_sub_into(z, nz, mc.qhalf, mc.wq);
      mp_add_into(z, nz, mc.q, mc.wq);
      uint32_t one = 1;
      mp_sub_into(z, nz, &one, 1);
      yneg = true;
    }
  }
  const int nq = nz - mc.wq + 1;
  if (!yzero) mp_div(z, nz, mc.qnorm, mc.wq, mc.qshift, un, qw);
  uint32_t* dst = out + (int64_t)st * mc.k * n + i;
  for (int j = 0; j < mc.k; ++j) {
    const Prime32Info inf = info[j];
    uint32_t r = yzero ? 0u : mp_mod_small(qw, nq, inf);
    if (yneg && r) r = inf.p - r;
    dst[(int64_t)j * n] = r;
  }
}

}  // namespace hefv

using namespace hefv;

extern "C" int hefv_decrypt_round(hefv_ctx* c, const uint32_t* acc, uint64_t* out, int64_t B,
                                   cudaStream_t st) {
  if (B <= 0) return 0;
  const int64_t total = B * c->n;
  k_decrypt_round<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(acc, out, B, mp_consts(c),
                                                                   c->d_info32);
  HEFV_LAUNCH_CHECK("k_decrypt_round");
  return 0;
}

extern "C" int hefv_mult_tensor_many(hefv_ctx* c, const uint32_t* a, int64_t a_stride,
                                     const uint32_t* b, int64_t b_stride, uint32_t* out3,
                                     uint32_t* scratch, int64_t B, void* stream) {
  if (!c || !c->fv_ready) return fail("hefv_mult_tensor: context without FV setup");
  if (c->a < 1 || c->wm < 1) return fail("hefv_mult_tensor: no auxiliary basis configured");
  if (B <= 0) return 0;
  if (B > 65535) return fail("hefv_mult_tensor: batch > 65535");
  cudaStream_t st = as_stream(stream);
  const int64_t n = c->n;
  const int64_t stack_a = (int64_t)c->a * n;
  const bool same = (a == b) && (a_stride == b_stride);
  const int nparts = same ? 2 : 4;
  uint32_t* L = scratch;                      // (B, nparts, a, N)
  uint32_t* T = scratch + B * 4 * stack_a;    // (B, 3, a, N)
  const MpConsts mc = mp_consts(c);
  {
    const int64_t tot = nparts * n;
    dim3 grid((unsigned)((tot + 127) / 128), (unsigned)B);
    k_mult_lift<<<grid, 128, 0, st>>>(a, a_stride, b, b_stride, nparts, L, mc, c->d_info32);
    HEFV_LAUNCH_CHECK("k_mult_lift");
  }
  if (int r = hefv_ntt_fwd32(c, L, L, nparts * B, c->a, c->k, 0, stream)) return r;
  {
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(148 * 8 / B + 1, (stack_a + 255) / 256));
    k_mult_tensor<<<dim3(gx, (unsigned)B), 256, 0, st>>>(L, same ? 1 : 0, T, mc, c->d_info32);
    HEFV_LAUNCH_CHECK("k_mult_tensor");
  }
  if (int r = hefv_ntt_inv32(c, T, T, 3 * B, c->a, c->k, 0, stream)) return r;
  {
    const int64_t tot = 3 * n;
    dim3 grid((unsigned)((tot + 63) / 64), (unsigned)B);
    k_mult_scale<<<grid, 64, 0, st>>>(T, out3, mc, c->d_info32);
    HEFV_LAUNCH_CHECK("k_mult_scale");
  }
  return 0;
}

extern "C" int hefv_mult_tensor(hefv_ctx* c, const uint32_t* a, const uint32_t* b,
                                uint32_t* out3, uint32_t* scratch, void* stream) {
  return hefv_mult_tensor_many(c, a, 0, b, 0, out3, scratch, 1, stream);
}
