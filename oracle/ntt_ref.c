/*
 * ORACLE (test infrastructure only -- never linked into the product).
 *
 * Plain-C restatement of the reference's CPU butterfly loop
 * (/root/reference/pkg/src/hepack/ntt.py:28-61, numba `_butterfly_kernel`):
 * an in-place iterative radix-2 Cooley-Tukey over the last axis of a
 * bit-reverse-permuted batch, per-stage twiddle tables concatenated
 * (lengths 1, 2, 4, ...), products reduced with a 32-bit Shoup companion
 * floor(w * 2^32 / p).  Valid for p < 2^31 with inputs in [0, p).
 * Used by oracle/fv_oracle.py as the CPU baseline's transform engine.
 */
#include <stdint.h>

void oracle_ct_stages(int64_t* x, int64_t batch, int64_t n, const int64_t* tw,
                      const int64_t* shoup, int64_t p) {
  for (int64_t b = 0; b < batch; ++b) {
    int64_t* row = x + b * n;
    int64_t half = 1, base = 0;
    while (half < n) {
      const int64_t step = half << 1;
      for (int64_t start = 0; start < n; start += step) {
        int64_t* lo = row + start;
        int64_t* hi = lo + half;
        for (int64_t j = 0; j < half; ++j) {
          const int64_t w = tw[base + j];
          const int64_t ws = shoup[base + j];
          const int64_t v = hi[j];
          const int64_t q = (v * ws) >> 32;
          int64_t t = v * w - q * p;
          if (t >= p) t -= p;
          const int64_t u = lo[j];
          int64_t s = u + t;
          if (s >= p) s -= p;
          int64_t d = u - t;
          if (d < 0) d += p;
          lo[j] = s;
          hi[j] = d;
        }
      }
      base += half;
      half = step;
    }
  }
}
