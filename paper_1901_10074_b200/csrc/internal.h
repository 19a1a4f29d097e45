// Internal (C++) view of a context.  Not part of the C-ABI: callers only
// see the opaque `hefv_ctx*` declared in include/hefv.h.
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "modarith.cuh"

namespace hefv {
// aux-basis key switch constants (ks_aux.cu)
struct KsaJ {
  uint2 c[3];      // (A / a_t) mod p_j, Shoup pair
  uint32_t e[4];   // (-v A) mod p_j, v = 0..3
};
struct KsaT {
  uint2 ninv[3];   // N^-1 (A / a_t)^-1 2^32 mod a_t, Shoup pair (last inverse stage)
  uint2 wn[3];     // psi_rev^-1[1] N^-1 (A / a_t)^-1 2^32 mod a_t, Shoup pair
  uint32_t qs[3];  // floor(2^46 / a_t): y * 2^14 / a_t = umulhi(y, qs)
};
}  // namespace hefv

struct hefv_ctx {
  int log_n = 0;
  int n = 0;
  // word-sized prime set: FV q primes first, then auxiliary primes
  int n32 = 0;
  std::vector<uint32_t> primes32;
  uint2* d_tw32 = nullptr;    // (n32, N) forward twiddles (psi^bitrev, shoup)
  uint2* d_itw32 = nullptr;   // (n32, N) inverse twiddles
  uint32_t* d_twm32 = nullptr;   // (n32, N) forward twiddles, Montgomery form
  uint32_t* d_itwm32 = nullptr;  // (n32, N) inverse twiddles, Montgomery form
  hefv::Prime32Info* d_info32 = nullptr;
  std::vector<hefv::Prime32Info> info32;
  // 64-bit prime set: plaintext modulus t (FV) or microbench primes
  int n64 = 0;
  std::vector<uint64_t> primes64;
  ulonglong2* d_tw64 = nullptr;
  ulonglong2* d_itw64 = nullptr;
  hefv::Prime64Info* d_info64 = nullptr;
  std::vector<hefv::Prime64Info> info64;
  // 64-bit Montgomery-free key-switch constants for 64-bit primes
  // (Shoup companions of keys are built on the fly)

  // ---- FV layer (set by hefv_fv_setup) ----
  bool fv_ready = false;
  int k = 0;           // q primes   = primes32[0, k)
  int a = 0;           // aux primes = primes32[k, k + a)
  int t_index = 0;     // t = primes64[t_index]
  uint64_t t = 0;
  int wq = 0, wm = 0;  // words of q and of the aux product M
  // device slot maps: slot -> device NTT index, device index -> slot (or -1)
  int32_t* d_slot_to_dev = nullptr;
  int32_t* d_dev_to_slot = nullptr;
  // multiprecision constants (little-endian 32-bit words), device copies
  uint32_t* d_mp = nullptr;  // one arena, offsets below
  size_t off_qhat = 0, off_qhatinv = 0, off_q = 0, off_qhalf = 0, off_qnorm = 0;
  size_t off_mhat = 0, off_mhatinv = 0, off_m = 0, off_mhalf = 0;
  int q_shift = 0;     // normalisation shift of q for long division
  uint32_t* d_delta = nullptr;   // Delta mod q_j (k)
  uint32_t* d_tmod = nullptr;    // t mod q_j (k)
  // aux-basis key switch (hefv_ks_aux_setup): three ~28-bit NTT primes at
  // primes32[ksa_base, ksa_base + 3)
  bool ksa_ready = false;
  bool ksa_shiftq = false;  // aux primes within 2^28 (1 + 1/16): CRT quotient terms by a shift
  int ksa_base = -1;
  hefv::KsaJ* d_ksa_j = nullptr;
  hefv::KsaT ksa_t{};
  // aux-basis 64-bit key switch (hefv_ks64_aux_setup): the T 32-bit primes of
  // the context are its aux primes
  int ks64a_T = 0;
  void* d_ks64a_t = nullptr;
  void* d_ks64a_j = nullptr;
  // key-switch accounting (hefv_ks_stats): calls and ciphertexts always;
  // with timing on, one CUDA event pair around every key-switch call
  int64_t ks_calls = 0, ks_cts = 0;
  bool ks_timing = false;
  std::vector<cudaEvent_t> ks_events;  // (begin, end) pairs
  // host -> device bytes copied by the library itself (plans, uploads)
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  // pinned staging buffers of the layer planner's host plans
  // (hefv_layer_rows): a buffer is reused once the copy recorded by its
  // event has completed, so calls on several streams never wait for each
  // other's queued work
  struct Stage {
    void* host = nullptr;
    size_t bytes = 0;
    cudaEvent_t done = nullptr;
  };
  std::vector<Stage> stages;
};

// switch-key handle of the object-level C-ABI (api.cu)
struct hefv_key {
  hefv_ctx* ctx = nullptr;
  uint32_t* body = nullptr;  // (k, k, N) [target j][digit i], device order, Montgomery form
  uint32_t* mask = nullptr;
  uint32_t* aux = nullptr;   // (3, 2k, k, N) aux-basis form, or null (per-prime key switch)
  bool owns = false;
};

namespace hefv {
void count_launch();
void set_error(const std::string& msg);
int fail(const std::string& msg);
int check_cuda(cudaError_t e, const char* where);
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
// key-switch call bracketing (context.cu): counts, and events when timing is on
void ks_begin(hefv_ctx* c, int64_t B, cudaStream_t st);
void ks_end(hefv_ctx* c, cudaStream_t st);
}  // namespace hefv

#define HEFV_CUDA(call)                                                     \
  do {                                                                      \
    cudaError_t _e = (call);                                                \
    if (_e != cudaSuccess) return hefv::check_cuda(_e, #call);              \
  } while (0)

#define HEFV_LAUNCH_CHECK(where)                                            \
  do {                                                                      \
    hefv::count_launch();                                                   \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess) return hefv::check_cuda(_e, where);              \
  } while (0)
