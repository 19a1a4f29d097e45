/*
 * A torch-free host of libhefv.so (test program for SURVEY.md 8b): plain C,
 * linked against libhefv.so and the CUDA runtime only.
 *
 *   hefv_host IN OUT
 *
 * IN (little-endian, written by tests/test_gpu_capi.py): the context setup
 * (primes, roots, CRT words -- what hepack's _FvContext precomputes,
 * fv.py:78-110), the relinearisation key and the Galois key of offset 1 in
 * the reference's stored form (SwitchKey body/mask, fv.py:67-72), two
 * ciphertexts as int64 (2, k, N) parts (FvCiphertext, fv.py:30-42) and one
 * slot vector.  OUT: rotate(a, 1), mult(a, b), add(a, b), add_plain(a, v),
 * cmult(a, v) as int64 (2, k, N) parts, in that order.
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "hefv.h"

static FILE* in_f;

static void* take(size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (!p || fread(p, 1, bytes, in_f) != bytes) {
    fprintf(stderr, "hefv_host: truncated input\n");
    exit(2);
  }
  return p;
}
static int64_t take_i64(void) {
  int64_t v;
  if (fread(&v, 8, 1, in_f) != 1) {
    fprintf(stderr, "hefv_host: truncated input\n");
    exit(2);
  }
  return v;
}
static void check(int rc, const char* what) {
  if (rc != 0) {
    fprintf(stderr, "hefv_host: %s failed (%d): %s\n", what, rc, hefv_last_error());
    exit(3);
  }
}

int main(int argc, char** argv) {
  if (argc != 3) {
    fprintf(stderr, "usage: hefv_host IN OUT\n");
    return 1;
  }
  in_f = fopen(argv[1], "rb");
  if (!in_f) return 1;
  const int64_t log_n = take_i64(), n32 = take_i64(), n64 = take_i64(), k = take_i64(),
                a = take_i64(), t_index = take_i64(), wq = take_i64(), wm = take_i64(),
                aux_base = take_i64();
  const int64_t n = (int64_t)1 << log_n;
  uint32_t* primes32 = take(4 * n32);
  uint32_t* psi32 = take(4 * n32);
  uint64_t* primes64 = take(8 * n64);
  uint64_t* psi64 = take(8 * n64);
  int32_t* slot_to_ev = take(4 * (n / 2));
  uint32_t* q = take(4 * wq);
  uint32_t* qhalf = take(4 * wq);
  uint32_t* qhat = take(4 * k * wq);
  uint32_t* qhat_inv = take(4 * k);
  uint32_t* m = take(4 * wm);
  uint32_t* mhalf = take(4 * wm);
  uint32_t* mhat = take(4 * a * wm);
  uint32_t* mhat_inv = take(4 * a);
  uint32_t* delta_mod = take(4 * k);
  const size_t key_words = (size_t)k * k * n, ct_words = (size_t)2 * k * n;
  int64_t* relin_body = take(8 * key_words);
  int64_t* relin_mask = take(8 * key_words);
  int64_t* rot_body = take(8 * key_words);
  int64_t* rot_mask = take(8 * key_words);
  int64_t* ct_a = take(8 * ct_words);
  int64_t* ct_b = take(8 * ct_words);
  uint64_t* slots = take(8 * (n / 2));
  fclose(in_f);

  hefv_ctx* ctx = NULL;
  check(hefv_ctx_create(&ctx, (uint32_t)log_n, (int32_t)n32, primes32, psi32, (int32_t)n64,
                        primes64, psi64),
        "hefv_ctx_create");
  check(hefv_fv_setup(ctx, (int32_t)k, (int32_t)a, (int32_t)t_index, slot_to_ev, (int32_t)wq, q,
                      qhalf, qhat, qhat_inv, (int32_t)wm, m, mhalf, mhat, mhat_inv, delta_mod),
        "hefv_fv_setup");
  if (aux_base >= 0) check(hefv_ks_aux_setup(ctx, (int32_t)aux_base), "hefv_ks_aux_setup");

  hefv_key *relin = NULL, *rot1 = NULL;
  check(hefv_key_upload(ctx, relin_body, relin_mask, &relin, NULL), "hefv_key_upload(relin)");
  check(hefv_key_upload(ctx, rot_body, rot_mask, &rot1, NULL), "hefv_key_upload(galois 1)");

  uint32_t *da, *db, *dout;
  check(hefv_ct_alloc(ctx, 2, &da), "hefv_ct_alloc");
  check(hefv_ct_alloc(ctx, 2, &db), "hefv_ct_alloc");
  check(hefv_ct_alloc(ctx, 2, &dout), "hefv_ct_alloc");
  check(hefv_ct_upload(ctx, ct_a, 2, da, NULL), "hefv_ct_upload(a)");
  check(hefv_ct_upload(ctx, ct_b, 2, db, NULL), "hefv_ct_upload(b)");
  uint64_t* dslots = NULL;
  if (cudaMalloc((void**)&dslots, 8 * (n / 2)) != cudaSuccess ||
      cudaMemcpy(dslots, slots, 8 * (n / 2), cudaMemcpyHostToDevice) != cudaSuccess) {
    fprintf(stderr, "hefv_host: slot upload failed\n");
    return 4;
  }

  FILE* out_f = fopen(argv[2], "wb");
  if (!out_f) return 1;
  int64_t* host = malloc(8 * ct_words);
  const uint32_t g1 = 3u;  /* 3^1 mod 2N: rotation by one slot (fv.py:427) */
  for (int op = 0; op < 5; ++op) {
    switch (op) {
      case 0: check(hefv_rotate(ctx, da, g1, rot1, dout, NULL), "hefv_rotate"); break;
      case 1: check(hefv_mult(ctx, da, db, relin, dout, NULL), "hefv_mult"); break;
      case 2: check(hefv_add(ctx, da, db, 2, dout, NULL), "hefv_add"); break;
      case 3: check(hefv_add_plain(ctx, da, 2, dslots, dout, NULL), "hefv_add_plain"); break;
      default: check(hefv_cmult(ctx, da, 2, dslots, dout, NULL), "hefv_cmult"); break;
    }
    check(hefv_ct_download(ctx, dout, 2, host, NULL), "hefv_ct_download");
    fwrite(host, 8, ct_words, out_f);
  }
  fclose(out_f);
  hefv_key_free(relin);
  hefv_key_free(rot1);
  hefv_ct_free(ctx, da);
  hefv_ct_free(ctx, db);
  hefv_ct_free(ctx, dout);
  cudaFree(dslots);
  hefv_ctx_destroy(ctx);
  printf("hefv_host: ok (k=%lld, N=%lld, launches=%llu)\n", (long long)k, (long long)n,
         (unsigned long long)hefv_launch_count());
  return 0;
}
