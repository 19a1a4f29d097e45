// Object-level C-ABI: ciphertext buffers, switch-key handles
// and the composite homomorphic operations of the reference's FvBackend,
// so that a host without torch drives the whole path through libhefv.so.
//
//   hefv_ct_alloc/free/upload/download   FvCiphertext parts (fv.py:30-42) <-> HBM
//   hefv_key_upload / wrap / free        SwitchKey (fv.py:67-72) -> device layout
//   hefv_encrypt_slots / decrypt_slots   _encrypt / _decrypt (fv.py:317-353)
//   hefv_add / add_plain / cmult         _add / _add_plain / _cmult (fv.py:355-375)
//   hefv_rotate                          one hop of _rotate (fv.py:417-432)
//   hefv_mult                            _mult + _relinearize (fv.py:377-415)
//
// Every composite op is a fixed sequence of the kernel-level entry points
// (the same sequence the Python backend issues), so its limbs are those of
// the reference.  Temporaries are stream-ordered (cudaMallocAsync /
// cudaFreeAsync on the caller's stream).
#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/hefv.h"
#include "internal.h"
#include "kcommon.cuh"

namespace hefv {

// Stream-ordered device temporary, released on scope exit.
struct DevTmp {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DevTmp() = default;
  DevTmp(const DevTmp&) = delete;
  DevTmp& operator=(const DevTmp&) = delete;
  ~DevTmp() {
    if (p) cudaFreeAsync(p, st);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

static int tmp_alloc(DevTmp& t, size_t bytes, cudaStream_t st) {
  t.st = st;
  HEFV_CUDA(cudaMallocAsync(&t.p, bytes > 0 ? bytes : 16, st));
  return 0;
}

static int need_fv(const hefv_ctx* c, const char* who) {
  if (!c) return fail(std::string(who) + ": null context");
  if (!c->fv_ready) return fail(std::string(who) + ": hefv_fv_setup has not been called");
  return 0;
}

// (k, k, N) natural evaluation order, canonical -> device order, Montgomery
// form: out[j][i][d] = in[j][i][bitrev(d)] * 2^32 mod p_j.
__global__ void k_key_import(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int k,
                             int log_n, const Prime32Info* __restrict__ info) {
  const int64_t total = ((int64_t)k * k) << log_n;
  const int n = 1 << log_n;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = g >> log_n;
    const int d = (int)(g & (n - 1));
    const int j = (int)(row / k);
    out[g] = mont_canon(in[(row << log_n) + brev_n(d, log_n)], info[j]);
  }
}

// (parts, k, N) int64 host residues -> uint32, each checked against p_j.
static int narrow_checked(const hefv_ctx* c, const int64_t* host, int64_t rows,
                          std::vector<uint32_t>& out, const char* who) {
  const int n = c->n;
  out.resize((size_t)rows * n);
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t p = c->primes32[r % c->k];
    const int64_t* src = host + r * n;
    uint32_t* dst = out.data() + r * n;
    for (int m = 0; m < n; ++m) {
      const int64_t v = src[m];
      if (v < 0 || v >= p) return fail(std::string(who) + ": residue outside [0, p_j)");
      dst[m] = (uint32_t)v;
    }
  }
  return 0;
}

// Key switch of one item (B = 1): out = KS_key(digits) + (adA0, adA1).
static int keyswitch_one(hefv_ctx* c, const hefv_key* key, const uint32_t* digits,
                         uint32_t galois, uint32_t* out0, uint32_t* out1, const uint32_t* adA0,
                         const uint32_t* adA1, cudaStream_t st) {
  if (key->aux) {
    DevTmp ws;
    if (int r = tmp_alloc(ws, (size_t)9 * c->k * c->n * 4, st)) return r;
    return hefv_keyswitch_aux(c, key->aux, digits, 0, nullptr, galois, out0, out1, 0, nullptr,
                              adA0, adA1, 0, nullptr, nullptr, 0, ws.as<uint32_t>(), 1, 1, st);
  }
  if (galois) return fail("keyswitch_one: the per-prime key switch needs materialised digits");
  return hefv_keyswitch(c, key->body, key->mask, digits, 0, out0, out1, 0, nullptr, adA0, adA1, 0,
                        nullptr, nullptr, 0, 1, st);
}

}  // namespace hefv

using namespace hefv;

extern "C" {

// ---- ciphertext buffers ------------------------------------------------------
int hefv_ct_alloc(hefv_ctx* c, int32_t nparts, uint32_t** out) {
  if (int r = need_fv(c, "hefv_ct_alloc")) return r;
  if (!out) return fail("hefv_ct_alloc: null out pointer");
  if (nparts < 1 || nparts > 3) return fail("hefv_ct_alloc: nparts must be 1..3");
  *out = nullptr;
  HEFV_CUDA(cudaMalloc(reinterpret_cast<void**>(out), (size_t)nparts * c->k * c->n * 4));
  return 0;
}

int hefv_transfer_stats(hefv_ctx* c, int64_t* h2d, int64_t* d2h) {
  if (!c) return fail("hefv_transfer_stats: null context");
  if (h2d) *h2d = c->h2d_bytes;
  if (d2h) *d2h = c->d2h_bytes;
  return 0;
}

int hefv_ct_free(hefv_ctx* c, uint32_t* ct) {
  (void)c;
  if (ct) HEFV_CUDA(cudaFree(ct));
  return 0;
}

int hefv_ct_upload(hefv_ctx* c, const int64_t* host, int32_t nparts, uint32_t* ct,
                   void* stream) {
  if (int r = need_fv(c, "hefv_ct_upload")) return r;
  if (!host || !ct) return fail("hefv_ct_upload: null pointer");
  if (nparts < 1 || nparts > 3) return fail("hefv_ct_upload: nparts must be 1..3");
  std::vector<uint32_t> words;
  if (int r = narrow_checked(c, host, (int64_t)nparts * c->k, words, "hefv_ct_upload")) return r;
  cudaStream_t st = as_stream(stream);
  HEFV_CUDA(cudaMemcpyAsync(ct, words.data(), words.size() * 4, cudaMemcpyHostToDevice, st));
  c->h2d_bytes += (int64_t)words.size() * 4;
  HEFV_CUDA(cudaStreamSynchronize(st));  // `words` is pageable and local
  return 0;
}

int hefv_ct_download(hefv_ctx* c, const uint32_t* ct, int32_t nparts, int64_t* host,
                     void* stream) {
  if (int r = need_fv(c, "hefv_ct_download")) return r;
  if (!host || !ct) return fail("hefv_ct_download: null pointer");
  if (nparts < 1 || nparts > 3) return fail("hefv_ct_download: nparts must be 1..3");
  const size_t words = (size_t)nparts * c->k * c->n;
  std::vector<uint32_t> buf(words);
  cudaStream_t st = as_stream(stream);
  HEFV_CUDA(cudaMemcpyAsync(buf.data(), ct, words * 4, cudaMemcpyDeviceToHost, st));
  c->d2h_bytes += (int64_t)words * 4;
  HEFV_CUDA(cudaStreamSynchronize(st));
  for (size_t i = 0; i < words; ++i) host[i] = buf[i];
  return 0;
}

// ---- switch keys -----------------------------------------------------------------
int hefv_key_upload(hefv_ctx* c, const int64_t* body, const int64_t* mask, hefv_key** out,
                    void* stream) {
  if (int r = need_fv(c, "hefv_key_upload")) return r;
  if (!body || !mask || !out) return fail("hefv_key_upload: null pointer");
  *out = nullptr;
  const int k = c->k;
  const size_t words = (size_t)k * k * c->n;
  cudaStream_t st = as_stream(stream);
  std::vector<uint32_t> hb, hm;
  // rows (j, i): residues mod p_j -- narrow_checked indexes primes by row % k,
  // so check per target prime j explicitly
  hb.resize(words);
  hm.resize(words);
  for (int j = 0; j < k; ++j) {
    const int64_t p = c->primes32[j];
    for (size_t q = 0; q < (size_t)k * c->n; ++q) {
      const size_t g = (size_t)j * k * c->n + q;
      const int64_t vb = body[g], vm = mask[g];
      if (vb < 0 || vb >= p || vm < 0 || vm >= p)
        return fail("hefv_key_upload: switch key residue outside [0, p_j)");
      hb[g] = (uint32_t)vb;
      hm[g] = (uint32_t)vm;
    }
  }
  hefv_key* key = new hefv_key();
  key->ctx = c;
  key->owns = true;
  auto cleanup = [&](int r) {
    hefv_key_free(key);
    return r;
  };
  if (cudaMalloc(reinterpret_cast<void**>(&key->body), words * 4) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&key->mask), words * 4) != cudaSuccess)
    return cleanup(fail("hefv_key_upload: out of device memory"));
  DevTmp raw;
  if (int r = tmp_alloc(raw, words * 4, st)) return cleanup(r);
  const unsigned grid = (unsigned)std::min<int64_t>(148 * 16, (int64_t)(words + 255) / 256);
  for (int part = 0; part < 2; ++part) {
    const std::vector<uint32_t>& h = part ? hm : hb;
    uint32_t* dst = part ? key->mask : key->body;
    if (cudaMemcpyAsync(raw.p, h.data(), words * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return cleanup(fail("hefv_key_upload: host-to-device copy failed"));
    c->h2d_bytes += (int64_t)words * 4;
    k_key_import<<<grid, 256, 0, st>>>(raw.as<uint32_t>(), dst, k, c->log_n, c->d_info32);
    count_launch();
    if (cudaGetLastError() != cudaSuccess) return cleanup(fail("hefv_key_upload: launch failed"));
  }
  if (c->ksa_ready) {
    int64_t aux_words = 0;
    if (int r = hefv_ks_aux_key_words(c, &aux_words)) return cleanup(r);
    if (cudaMalloc(reinterpret_cast<void**>(&key->aux), (size_t)aux_words * 4) != cudaSuccess)
      return cleanup(fail("hefv_key_upload: out of device memory (aux key)"));
    if (int r = hefv_ks_aux_key(c, key->body, key->mask, key->aux, st)) return cleanup(r);
  }
  if (cudaStreamSynchronize(st) != cudaSuccess)  // hb / hm are pageable and local
    return cleanup(fail("hefv_key_upload: stream synchronisation failed"));
  *out = key;
  return 0;
}

int hefv_key_wrap(hefv_ctx* c, const uint32_t* body, const uint32_t* mask, const uint32_t* aux,
                  hefv_key** out) {
  if (int r = need_fv(c, "hefv_key_wrap")) return r;
  if (!body || !mask || !out) return fail("hefv_key_wrap: null pointer");
  if (c->ksa_ready && !aux) return fail("hefv_key_wrap: this context needs the aux-basis key form");
  hefv_key* key = new hefv_key();
  key->ctx = c;
  key->body = const_cast<uint32_t*>(body);
  key->mask = const_cast<uint32_t*>(mask);
  key->aux = c->ksa_ready ? const_cast<uint32_t*>(aux) : nullptr;
  key->owns = false;
  *out = key;
  return 0;
}

int hefv_key_free(hefv_key* key) {
  if (!key) return 0;
  if (key->owns) {
    cudaFree(key->body);
    cudaFree(key->mask);
    cudaFree(key->aux);
  }
  delete key;
  return 0;
}

// ---- encryption / decryption ------------------------------------------------------
int hefv_encrypt_slots(hefv_ctx* c, const uint32_t* pk_ntt, const int8_t* u, const int8_t* e1,
                       const int8_t* e2, const uint64_t* slots, uint32_t* out, int64_t B,
                       void* stream) {
  if (int r = need_fv(c, "hefv_encrypt_slots")) return r;
  if (B <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  DevTmp poly, dm;
  if (int r = tmp_alloc(poly, (size_t)B * c->n * 8, st)) return r;
  if (int r = tmp_alloc(dm, (size_t)B * c->k * c->n * 4, st)) return r;
  if (int r = hefv_encode(c, slots, poly.as<uint64_t>(), B, st)) return r;
  if (int r = hefv_plain_to_rns(c, poly.as<uint64_t>(), dm.as<uint32_t>(), B, 0, 0, 0, st)) return r;
  return hefv_encrypt(c, pk_ntt, u, e1, e2, dm.as<uint32_t>(), out, B, st);
}

int hefv_decrypt_slots(hefv_ctx* c, const uint32_t* ct, int32_t nparts, const uint32_t* s_ntt,
                       const uint32_t* s2_ntt, uint64_t* slots, int64_t B, void* stream) {
  if (int r = need_fv(c, "hefv_decrypt_slots")) return r;
  if (B <= 0) return 0;
  cudaStream_t st = as_stream(stream);
  DevTmp poly, scratch;
  if (int r = tmp_alloc(poly, (size_t)B * c->n * 8, st)) return r;
  if (int r = tmp_alloc(scratch, (size_t)B * c->k * c->n * 4, st)) return r;
  if (int r = hefv_decrypt(c, ct, nparts, s_ntt, s2_ntt, poly.as<uint64_t>(),
                           scratch.as<uint32_t>(), B, st))
    return r;
  return hefv_decode(c, poly.as<uint64_t>(), slots, B, st);
}

// ---- linear ops -----------------------------------------------------------------------
int hefv_add(hefv_ctx* c, const uint32_t* a, const uint32_t* b, int32_t nparts, uint32_t* out,
             void* stream) {
  if (int r = need_fv(c, "hefv_add")) return r;
  if (nparts < 1 || nparts > 3) return fail("hefv_add: nparts must be 1..3");
  return hefv_elementwise(c, 0, a, b, nullptr, out, nparts, nparts, 0, stream);
}

int hefv_add_plain(hefv_ctx* c, const uint32_t* ct, int32_t nparts, const uint64_t* slots,
                   uint32_t* out, void* stream) {
  if (int r = need_fv(c, "hefv_add_plain")) return r;
  if (nparts < 1 || nparts > 3) return fail("hefv_add_plain: nparts must be 1..3");
  cudaStream_t st = as_stream(stream);
  const size_t stack = (size_t)c->k * c->n;
  DevTmp poly, dm;
  if (int r = tmp_alloc(poly, (size_t)c->n * 8, st)) return r;
  if (int r = tmp_alloc(dm, stack * 4, st)) return r;
  if (int r = hefv_encode(c, slots, poly.as<uint64_t>(), 1, st)) return r;
  // Delta * m with m uncentred (_delta_m, fv.py:296-310), added to c0 only
  if (int r = hefv_plain_to_rns(c, poly.as<uint64_t>(), dm.as<uint32_t>(), 1, 0, 0, 0, st)) return r;
  if (nparts > 1 && out != ct)
    HEFV_CUDA(cudaMemcpyAsync(out + stack, ct + stack, (nparts - 1) * stack * 4,
                              cudaMemcpyDeviceToDevice, st));
  return hefv_elementwise(c, 0, ct, dm.as<uint32_t>(), nullptr, out, 1, 1, 0, st);
}

int hefv_cmult(hefv_ctx* c, const uint32_t* ct, int32_t nparts, const uint64_t* slots,
               uint32_t* out, void* stream) {
  if (int r = need_fv(c, "hefv_cmult")) return r;
  if (nparts < 1 || nparts > 3) return fail("hefv_cmult: nparts must be 1..3");
  cudaStream_t st = as_stream(stream);
  DevTmp poly, m;
  if (int r = tmp_alloc(poly, (size_t)c->n * 8, st)) return r;
  if (int r = tmp_alloc(m, (size_t)c->k * c->n * 4, st)) return r;
  if (int r = hefv_encode(c, slots, poly.as<uint64_t>(), 1, st)) return r;
  // centred m, NTT, Montgomery form (fv.py:366-370)
  if (int r = hefv_plain_to_rns(c, poly.as<uint64_t>(), m.as<uint32_t>(), 1, 1, 1, 1, st)) return r;
  return hefv_mul_plain(c, ct, m.as<uint32_t>(), out, 1, nparts, 1, st);
}

// ---- rotation hop / multiplication ---------------------------------------------------------
int hefv_rotate(hefv_ctx* c, const uint32_t* ct, uint32_t galois_elt, const hefv_key* key,
                uint32_t* out, void* stream) {
  if (int r = need_fv(c, "hefv_rotate")) return r;
  if (!key || key->ctx != c) return fail("hefv_rotate: key belongs to another context");
  if ((galois_elt & 1u) == 0) return fail("hefv_rotate: galois element must be odd");
  cudaStream_t st = as_stream(stream);
  const size_t stack = (size_t)c->k * c->n;
  DevTmp sig;
  if (key->aux) {
    // sigma(c0) materialised; sigma(c1) applied inside the key switch's digit load
    if (int r = tmp_alloc(sig, stack * 4, st)) return r;
    if (int r = hefv_automorph(c, ct, 0, nullptr, sig.as<uint32_t>(), 1, galois_elt, 1, st)) return r;
    return keyswitch_one(c, key, ct + stack, galois_elt, out, out + stack, sig.as<uint32_t>(),
                         nullptr, st);
  }
  if (int r = tmp_alloc(sig, 2 * stack * 4, st)) return r;
  if (int r = hefv_automorph(c, ct, 0, nullptr, sig.as<uint32_t>(), 2, galois_elt, 1, st)) return r;
  return keyswitch_one(c, key, sig.as<uint32_t>() + stack, 0, out, out + stack,
                       sig.as<uint32_t>(), nullptr, st);
}

int hefv_mult(hefv_ctx* c, const uint32_t* a, const uint32_t* b, const hefv_key* relin,
              uint32_t* out, void* stream) {
  if (int r = need_fv(c, "hefv_mult")) return r;
  if (!relin || relin->ctx != c) return fail("hefv_mult: key belongs to another context");
  cudaStream_t st = as_stream(stream);
  const size_t stack = (size_t)c->k * c->n;
  DevTmp out3, scratch;
  if (int r = tmp_alloc(out3, 3 * stack * 4, st)) return r;
  if (int r = tmp_alloc(scratch, (size_t)7 * c->a * c->n * 4, st)) return r;
  if (int r = hefv_mult_tensor(c, a, b, out3.as<uint32_t>(), scratch.as<uint32_t>(), st)) return r;
  // relinearisation (fv.py:411-415): (t0, t1) + KS_relin(t2)
  uint32_t* t = out3.as<uint32_t>();
  return keyswitch_one(c, relin, t + 2 * stack, 0, out, out + stack, t, t + stack, st);
}

}  // extern "C"
