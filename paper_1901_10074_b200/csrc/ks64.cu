// RNS-limb key switch over 64-bit primes (config 4 microbench: L primes of
// 50-62 bits, N up to 2^16).  Same algorithm as _keyswitch_apply (reference
// fv.py:205-217, which takes the object-dtype path for such primes):
//   digits D[i][j] = NTT_j(c_i mod p_j); acc_j = sum_i D[i][j] * key[j][i];
//   (d0_j, d1_j) = iNTT_j(acc0_j, acc1_j).
// The polynomials (up to 512 KB each) exceed a CTA's shared memory, so the
// pipeline is three stages through HBM: replicate+reduce the digits, the
// batched 64-bit NTT (ntt_kernels.cu), a fused Montgomery MAC over the L
// digits, and the batched inverse NTT in place.
#include "../../include/hefv.h"
#include "internal.h"
#include "kcommon.cuh"

namespace hefv {

// scratch[b][i][j][n] = digits[b][i][n] mod p_j
__global__ void k_ks64_replicate(const uint64_t* __restrict__ digits, uint64_t* __restrict__ scr,
                                 int L, int log_n, int64_t total,
                                 const Prime64Info* __restrict__ info) {
  const int64_t n = 1ll << log_n;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = g & (n - 1);
    const int64_t r = g >> log_n;  // (b, i, j)
    const int j = (int)(r % L);
    const int64_t bi = r / L;      // b * L + i
    const uint64_t v = digits[(bi << log_n) + w];
    const uint64_t p = info[j].p;
    scr[g] = v >= p ? v % p : v;
  }
}

// out[b][part][j][n] = sum_i scr[b][i][j][n] * key_part[j][i][n]   (lazy, then canonical)
__global__ void k_ks64_mac(const uint64_t* __restrict__ scr, const uint64_t* __restrict__ kbody,
                           const uint64_t* __restrict__ kmask, uint64_t* __restrict__ out, int L,
                           int log_n, int64_t total, const Prime64Info* __restrict__ info) {
  const int64_t n = 1ll << log_n;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {  // g over (b, j, n)
    const int64_t w = g & (n - 1);
    const int64_t r = g >> log_n;
    const int j = (int)(r % L);
    const int64_t b = r / L;
    const Prime64Info inf = info[j];
    const uint64_t p2 = 2 * inf.p;
    uint64_t a0 = 0, a1 = 0;
    for (int i = 0; i < L; ++i) {
      const uint64_t d = scr[(((b * L + i) * L + j) << log_n) + w];
      const int64_t ko = (((int64_t)j * L + i) << log_n) + w;
      a0 += mont_mul64_lazy(d, kbody[ko], inf.p, inf.pinv_neg);
      a1 += mont_mul64_lazy(d, kmask[ko], inf.p, inf.pinv_neg);
      a0 = a0 >= p2 ? a0 - p2 : a0;
      a1 = a1 >= p2 ? a1 - p2 : a1;
    }
    a0 = a0 >= inf.p ? a0 - inf.p : a0;
    a1 = a1 >= inf.p ? a1 - inf.p : a1;
    out[(((b * 2 + 0) * L + j) << log_n) + w] = a0;
    out[(((b * 2 + 1) * L + j) << log_n) + w] = a1;
  }
}

// x -> x * 2^64 mod p (Montgomery form) over (rows, L, N)
__global__ void k_to_mont64(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int L,
                            int log_n, int64_t total, const Prime64Info* __restrict__ info) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)((g >> log_n) % L);
    const Prime64Info inf = info[j];
    uint64_t v = mont_mul64_lazy(in[g] % inf.p, inf.r2, inf.p, inf.pinv_neg);
    out[g] = v >= inf.p ? v - inf.p : v;
  }
}

}  // namespace hefv

using namespace hefv;

extern "C" {

int hefv_to_montgomery64(hefv_ctx* c, const uint64_t* in, uint64_t* out, int64_t rows,
                         void* stream) {
  if (!c || c->n64 < 1) return fail("hefv_to_montgomery64: context has no 64-bit primes");
  const int L = c->n64;
  const int64_t total = rows * L * (int64_t)c->n;
  if (total <= 0) return 0;
  k_to_mont64<<<148 * 16, 256, 0, as_stream(stream)>>>(in, out, L, c->log_n, total, c->d_info64);
  HEFV_LAUNCH_CHECK("k_to_mont64");
  return 0;
}

int hefv_keyswitch64(hefv_ctx* c, const uint64_t* kbody, const uint64_t* kmask,
                     const uint64_t* digits, uint64_t* out, uint64_t* scratch, int64_t B,
                     void* stream) {
  if (!c || c->n64 < 1) return fail("hefv_keyswitch64: context has no 64-bit primes");
  if (B <= 0) return 0;
  const int L = c->n64;
  cudaStream_t st = as_stream(stream);
  const int64_t n = c->n;
  const int64_t tot_rep = B * L * L * n;
  k_ks64_replicate<<<148 * 16, 256, 0, st>>>(digits, scratch, L, c->log_n, tot_rep, c->d_info64);
  HEFV_LAUNCH_CHECK("k_ks64_replicate");
  if (int r = hefv_ntt_fwd64(c, scratch, scratch, B * L, L, 0, 0, stream)) return r;
  const int64_t tot_mac = B * L * n;
  k_ks64_mac<<<148 * 16, 256, 0, st>>>(scratch, kbody, kmask, out, L, c->log_n, tot_mac,
                                       c->d_info64);
  HEFV_LAUNCH_CHECK("k_ks64_mac");
  return hefv_ntt_inv64(c, out, out, 2 * B, L, 0, 0, stream);
}

}  // extern "C"
