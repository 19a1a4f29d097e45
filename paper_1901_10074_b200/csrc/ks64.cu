// RNS-limb key switch over 64-bit primes (config 4 microbench: L primes of
// 50-62 bits, N up to 2^16).  Same algorithm as _keyswitch_apply (reference
// fv.py:205-217, which takes the object-dtype path for such primes):
//   digits D[i][j] = NTT_j(c_i mod p_j); acc_j = sum_i D[i][j] * key[j][i];
//   (d0_j, d1_j) = iNTT_j(acc0_j, acc1_j).
// The polynomials (up to 512 KB each) exceed a CTA's shared memory, so the
// pipeline is three stages through HBM: the batched 64-bit NTT of every digit
// row under every prime (ntt_kernels.cu, reading each row L times with the
// reduction mod p_j fused into the load), a Montgomery MAC over the L digits,
// and the batched inverse NTT in place.
#include "../../include/hefv.h"
#include "internal.h"
#include "kcommon.cuh"

int hefv_ntt64_fwd_rows(hefv_ctx* c, const uint64_t* in, uint64_t* out, int64_t rows,
                        cudaStream_t st);

namespace hefv {

// out[b][part][j][n] = sum_i scr[b][i][j][n] * key_part[j][i][n]   (lazy, then canonical)
// grid: x = point blocks, y = (b, j) row; 32-bit indexing inside a row.
__global__ void __launch_bounds__(256)
    k_ks64_mac(const uint64_t* __restrict__ scr, const uint64_t* __restrict__ kbody,
               const uint64_t* __restrict__ kmask, uint64_t* __restrict__ out, int L, int log_n,
               const Prime64Info* __restrict__ info) {
  const int n = 1 << log_n;
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n) return;
  const int row = blockIdx.y;  // b * L + j
  const int b = row / L, j = row - b * L;
  const uint64_t p = info[j].p, pinv_neg = info[j].pinv_neg, p2 = 2 * p;
  const uint64_t* d = scr + ((size_t)b * L * L + j) * n + w;  // digit i at + i * L * n
  const uint64_t* kb = kbody + (size_t)j * L * n + w;         // digit i at + i * n
  const uint64_t* km = kmask + (size_t)j * L * n + w;
  uint64_t a0 = 0, a1 = 0;
  for (int i = 0; i < L; ++i) {
    const uint64_t di = __ldg(d + (size_t)i * L * n);
    a0 += mont_mul64_lazy(di, __ldg(kb + (size_t)i * n), p, pinv_neg);
    a1 += mont_mul64_lazy(di, __ldg(km + (size_t)i * n), p, pinv_neg);
    a0 = a0 >= p2 ? a0 - p2 : a0;
    a1 = a1 >= p2 ? a1 - p2 : a1;
  }
  a0 = a0 >= p ? a0 - p : a0;
  a1 = a1 >= p ? a1 - p : a1;
  out[((size_t)(b * 2 + 0) * L + j) * n + w] = a0;
  out[((size_t)(b * 2 + 1) * L + j) * n + w] = a1;
}

// x -> x * 2^64 mod p (Montgomery form) over (rows, L, N)
__global__ void k_to_mont64(const uint64_t* __restrict__ in, uint64_t* __restrict__ out, int L,
                            int log_n, int64_t total, const Prime64Info* __restrict__ info) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)((g >> log_n) % L);
    const Prime64Info inf = info[j];
    const uint64_t x = in[g];
    uint64_t v = mont_mul64_lazy(x >= inf.p ? barrett64(x, inf.p, inf.mu) : x, inf.r2, inf.p,
                                 inf.pinv_neg);
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
  if (B * L > 65535) return fail("hefv_keyswitch64: batch too large");
  // digit rows (b, i) -> NTT_j(c_i mod p_j) for every j, straight from the
  // digit rows (no reduced copies)
  if (int r = hefv_ntt64_fwd_rows(c, digits, scratch, B * L, st)) return r;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)(B * L));
  k_ks64_mac<<<grid, 256, 0, st>>>(scratch, kbody, kmask, out, L, c->log_n, c->d_info64);
  HEFV_LAUNCH_CHECK("k_ks64_mac");
  return hefv_ntt_inv64(c, out, out, 2 * B, L, 0, 0, stream);
}

}  // extern "C"
