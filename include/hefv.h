/*
 * hefv.h -- C-ABI of the B200-native RNS/FV hot path (libhefv.so).
 *
 * Drop-in boundary for the reference `hepack` FV backend:
 * every entry point below replaces one CPU routine of the reference, cited
 * as /root/reference/pkg/src/hepack/<file>:<line>.  Signatures use only
 * plain pointers, sizes and an opaque context; device pointers are CUDA
 * global-memory addresses (the Python host side allocates them with torch),
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Conventions
 *   - A "stack" is (k, N) uint32 residues, limb-major, values in [0, p_j):
 *     the reference's `np.int64` (k, N) coefficient arrays (fv.py:30-42)
 *     narrowed to 32 bits.  A ciphertext is (parts, k, N); a batch of B
 *     ciphertexts is (B, parts, k, N).
 *   - "device NTT order" is the bit-reversed order of the reference's
 *     natural evaluation order: dev[i] = NttPrime.fwd(a)[bitrev(i)]
 *     (ntt.py:145-147).  Switch keys and cached key material live in that
 *     order, in Montgomery form (x * 2^32 mod p) where noted.
 *   - Every function returns 0 on success and a negative code on error;
 *     hefv_last_error() returns a thread-local message.  Launch errors are
 *     reported synchronously; kernels are asynchronous on `stream`.
 */
#ifndef HEFV_H
#define HEFV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hefv_ctx hefv_ctx;

/* ---- housekeeping ------------------------------------------------------ */
const char* hefv_last_error(void);
int hefv_abi_version(void);
/* Number of kernels this library has launched (all contexts, process-wide). */
uint64_t hefv_launch_count(void);

/* Context: NTT tables for a set of word-sized primes (2^28 < p < 2^30) and a
 * set of 64-bit primes (p < 2^62), ring dimension N = 2^log_n, 1 <= log_n <= 16
 * (the FV entry points need 4 <= log_n <= 14).
 * Replaces NttPrime.__init__ (ntt.py:149-172) for every prime of
 * _FvContext.__init__ (fv.py:83, fv.py:95, fv.py:101).  psi is the primitive
 * 2N-th root the reference picks (g^((p-1)/2N), g the smallest generator). */
int hefv_ctx_create(hefv_ctx** out, uint32_t log_n, int32_t n32, const uint32_t* primes32,
                    const uint32_t* psi32, int32_t n64, const uint64_t* primes64,
                    const uint64_t* psi64);
void hefv_ctx_destroy(hefv_ctx* ctx);

/* ---- negacyclic NTT (K1/K2/K3) -----------------------------------------
 * data (batch, nprimes, N); polynomial (b, i) uses prime prime_base + i of
 * the 32-bit (or 64-bit) set.  natural = 1 uses the reference's natural
 * evaluation order, 0 the device order.  Inputs of the forward transform
 * may be any word (reduced mod p on load); inputs of the inverse must be
 * canonical.  Outputs are canonical.
 * Replace NttPrime.fwd (ntt.py:216-219) and NttPrime.inv (ntt.py:221-224). */
int hefv_ntt_fwd32(hefv_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t batch,
                   int32_t nprimes, int32_t prime_base, int32_t natural, void* stream);
int hefv_ntt_inv32(hefv_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t batch,
                   int32_t nprimes, int32_t prime_base, int32_t natural, void* stream);
int hefv_ntt_fwd64(hefv_ctx* ctx, const uint64_t* in, uint64_t* out, int64_t batch,
                   int32_t nprimes, int32_t prime_base, int32_t natural, void* stream);
int hefv_ntt_inv64(hefv_ctx* ctx, const uint64_t* in, uint64_t* out, int64_t batch,
                   int32_t nprimes, int32_t prime_base, int32_t natural, void* stream);

/* Pointwise product of canonical residue rows: out = a * b mod p, data
 * (batch, nprimes, N) as above (words of 4 bytes, or 8 when wide = 1).
 * The middle step of NttPrime.negacyclic_mul (ntt.py:226-227). */
int hefv_pointwise_mul(hefv_ctx* ctx, int32_t wide, const void* a, const void* b, void* out,
                       int64_t batch, int32_t nprimes, int32_t prime_base, void* stream);

/* ---- FV layer setup ------------------------------------------------------
 * k q-primes = 32-bit primes [0, k), a auxiliary primes = [k, k + a),
 * t = 64-bit prime t_index.  slot_to_ev: (N/2) natural evaluation index of
 * every slot (fv.py:102-109).  Multiprecision constants are little-endian
 * 32-bit words: q (wq words), floor(q/2), qhat_i = q/q_i (k x wq),
 * qhat_inv_i = (q/q_i)^-1 mod q_i; the same for the auxiliary product M
 * (wm words).  delta_mod_j = floor(q/t) mod q_j (fv.py:86-87). */
int hefv_fv_setup(hefv_ctx* ctx, int32_t k, int32_t a, int32_t t_index,
                  const int32_t* slot_to_ev, int32_t wq, const uint32_t* q_words,
                  const uint32_t* qhalf_words, const uint32_t* qhat_words,
                  const uint32_t* qhat_inv, int32_t wm, const uint32_t* m_words,
                  const uint32_t* mhalf_words, const uint32_t* mhat_words,
                  const uint32_t* mhat_inv, const uint32_t* delta_mod);

/* ---- batching: encode / decode (fv.py:280-289) ---------------------------
 * slots: (B, N/2) uint64 residues mod t; poly: (B, N) uint64 in [0, t). */
int hefv_encode(hefv_ctx* ctx, const uint64_t* slots, uint64_t* poly, int64_t B, void* stream);
int hefv_decode(hefv_ctx* ctx, const uint64_t* poly, uint64_t* slots, int64_t B, void* stream);
/* Sparse encode for the layer planner: plaintext p has entries
 * [ptr[p], ptr[p+1]) of (slot, value mod t); others are zero. */
int hefv_encode_sparse(hefv_ctx* ctx, const int32_t* ptr, const int32_t* slot_idx,
                       const uint64_t* vals, uint64_t* poly, int64_t P, void* stream);

/* Plaintext poly (B, N) in [0, t) -> RNS stack (B, k, N).
 * mode 0: Delta * m mod q_j with m uncentred (_delta_m, fv.py:296-310);
 * mode 1: centred m mod q_j (_centered_plain + `m % tr.p`, fv.py:291-294,
 *         fv.py:366-370).  to_ntt = 1 additionally applies the forward NTT
 *         (device order); montgomery = 1 stores x * 2^32 mod q_j. */
int hefv_plain_to_rns(hefv_ctx* ctx, const uint64_t* poly, uint32_t* out, int64_t B,
                      int32_t mode, int32_t to_ntt, int32_t montgomery, void* stream);

/* Signed small polynomials (B, N) int8 -> (B, k, N) residues, optionally NTT
 * (device order) and Montgomery form.  Replaces _FvContext.to_rns (fv.py:119-122). */
int hefv_small_to_rns(hefv_ctx* ctx, const int8_t* small, uint32_t* out, int64_t B,
                      int32_t to_ntt, int32_t montgomery, void* stream);

/* ---- elementwise ----------------------------------------------------------
 * op 0: out = a + b; 1: out = a - b; 2: out = a * b (both canonical, plain
 * form); 3: out = -(a*b + c) (keygen body); over `rows` stacks of (k, N).
 * b_rows/c_rows = 1 broadcasts one stack.  Replaces _FvContext.add/neg
 * (fv.py:131-135) and the pointwise products of fv.py:212-213, 330. */
int hefv_elementwise(hefv_ctx* ctx, int32_t op, const uint32_t* a, const uint32_t* b,
                     const uint32_t* c, uint32_t* out, int64_t rows, int64_t b_rows,
                     int64_t c_rows, void* stream);
/* out stack = montgomery form of a (x * 2^32 mod p). */
int hefv_to_montgomery(hefv_ctx* ctx, const uint32_t* a, uint32_t* out, int64_t rows,
                       void* stream);

/* ---- encryption / decryption (fv.py:317-353) ----------------------------
 * pk_ntt: (2, k, N) NTT(pk) in device order, Montgomery form.  u, e1, e2:
 * (B, N) int8 drawn on the host by the reference's Generator calls.  dm:
 * (B, k, N) Delta*m.  out: (B, 2, k, N). */
int hefv_encrypt(hefv_ctx* ctx, const uint32_t* pk_ntt, const int8_t* u, const int8_t* e1,
                 const int8_t* e2, const uint32_t* dm, uint32_t* out, int64_t B, void* stream);
/* ct: (B, nparts, k, N), nparts in {2, 3}; s_ntt, s2_ntt: (k, N) device
 * order, Montgomery form.  out: (B, N) uint64 plaintext poly mod t
 * (decrypt_poly, fv.py:337-349).  scratch: (B, k, N) uint32. */
int hefv_decrypt(hefv_ctx* ctx, const uint32_t* ct, int32_t nparts, const uint32_t* s_ntt,
                 const uint32_t* s2_ntt, uint64_t* out, uint32_t* scratch, int64_t B,
                 void* stream);

/* ---- ciphertext x plaintext (fv.py:364-375) --------------------------------
 * out[b][part] = iNTT(NTT(ct[b][part]) * m_ntt[b or 0]) for each q prime;
 * m_ntt: (B or 1, k, N) device order, Montgomery form. */
int hefv_mul_plain(hefv_ctx* ctx, const uint32_t* ct, const uint32_t* m_ntt, uint32_t* out,
                   int64_t B, int32_t nparts, int32_t m_broadcast, void* stream);
/* Layer planner MAC: x_ntt (kin, 2, k, N) Montgomery device-order NTTs of the
 * input ciphertexts; m_ntt (P, k, N) plain NTTs; row r sums plaintexts
 * [row_ptr[r], row_ptr[r+1]) each against input ciphertext plain_seg[p];
 * out (R, 2, k, N) coefficient domain.  Equals the reference's segment
 * cmult + add chain (inference.py:304-311). */
int hefv_rows_mac(hefv_ctx* ctx, const uint32_t* x_ntt, const uint32_t* m_ntt,
                  const int32_t* row_ptr, const int32_t* plain_seg, uint32_t* out, int64_t R,
                  void* stream);
/* The same MAC with a plaintext index per tap: row r sums, over taps t in
 * [row_ptr[r], row_ptr[r+1]), m_ntt[tap_plain[t]] * x_ntt[tap_src[t]].  Used
 * by the interleaved (per-pixel broadcast) layers, inference.py:406-428:
 * every cmult by np.full(width, w) shares the plaintext of its weight value,
 * and the row's cmult + add chain is one NTT-domain sum (linear, exact). */
int hefv_rows_mac_indexed(hefv_ctx* ctx, const uint32_t* x_ntt, const uint32_t* m_ntt,
                          const int32_t* row_ptr, const int32_t* tap_src,
                          const int32_t* tap_plain, uint32_t* out, int64_t R, void* stream);

/* ---- rotations (fv.py:157-173, fv.py:417-432) -----------------------------
 * Galois automorphism x -> x^g (g odd) of `nparts` parts of B ciphertexts:
 * source ciphertext b is in + slot[b] * in_stride (slot may be NULL);
 * out is dense (B, nparts, k, N). */
int hefv_automorph(hefv_ctx* ctx, const uint32_t* in, int64_t in_stride, const int32_t* slot,
                   uint32_t* out, int32_t nparts, uint32_t galois_elt, int64_t B, void* stream);

/* RNS-limb key switch (K4, fv.py:205-217), batched over B ciphertexts that
 * share one switch key.  kbody/kmask: (k, k, N) = [target prime j][digit i],
 * device NTT order, Montgomery form.  digits of item b: digits + b*dig_stride
 * ((k, N) coefficient limbs).  Epilogue, per part p in {0,1}:
 *   out_p[slot b] = d_p + adA_p[b] + adB_p[slot b]     (mod q_j)
 * with out/adB at ptr + slot[b]*stride (slot may be NULL) and adA dense;
 * any adA/adB pointer may be NULL; adB may alias out. */
int hefv_keyswitch(hefv_ctx* ctx, const uint32_t* kbody, const uint32_t* kmask,
                   const uint32_t* digits, int64_t dig_stride, uint32_t* out0, uint32_t* out1,
                   int64_t out_stride, const int32_t* slot, const uint32_t* adA0,
                   const uint32_t* adA1, int64_t adA_stride, const uint32_t* adB0,
                   const uint32_t* adB1, int64_t adB_stride, int64_t B, void* stream);

/* Switch-key generation for one digit i (fv.py:176-202), NTT domain:
 *   kbody[j][i] = g_i,j * target[j] - (A_j * s[j] + E_j),  kmask[j][i] = A_j
 * with A = NTT(a_i), E = NTT(e_i); a_i (k, N) uniform residues, e_i (N) int8;
 * s_ntt, target_ntt canonical device order; gadget_i: (k) g_i mod q_j.
 * Outputs are written in Montgomery form. */
int hefv_keygen_digit(hefv_ctx* ctx, const uint32_t* a_i, const int8_t* e_i, int32_t digit,
                      const uint32_t* gadget_i, const uint32_t* s_ntt,
                      const uint32_t* target_ntt, uint32_t* kbody, uint32_t* kmask,
                      void* stream);

/* ---- ciphertext x ciphertext (K8, fv.py:377-409) --------------------------
 * Exact BFV tensor with multiprecision CRT lift and t/q rounding.
 * a, b: (2, k, N) each (b may equal a).  out3: (3, k, N) -- the unrelinearised
 * parts; scratch: at least 7 * a * N uint32 (aux stacks). */
int hefv_mult_tensor(hefv_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out3,
                     uint32_t* scratch, void* stream);
/* Batched tensor step of B products a[i] x b[i]: a[i] = a + i * a_stride,
 * b[i] = b + i * b_stride (uint32 words), out3 (B, 3, k, N), scratch
 * B * 7 * a * N words.  a == b with equal strides are squares (only the two
 * parts of each operand are lifted). */
int hefv_mult_tensor_many(hefv_ctx* ctx, const uint32_t* a, int64_t a_stride, const uint32_t* b,
                          int64_t b_stride, uint32_t* out3, uint32_t* scratch, int64_t B,
                          void* stream);

/* ---- layer planner helpers ---------------------------------------------------
 * out[dst] (+)= sum of rows[r] for r in [seg[m], seg[m+1]) for m < M, with
 * dst = seg_out[m]; rows (R, 2, k, N); out (nout, 2, k, N).  accumulate = 1
 * adds into out, 0 overwrites (inference.py:333-338). */
int hefv_accumulate_rows(hefv_ctx* ctx, const uint32_t* rows, const int32_t* seg,
                         const int32_t* seg_out, uint32_t* out, int32_t M, int32_t accumulate,
                         void* stream);
/* rows[slot[i]] part 0 += add[i] (i < P): the batched add_plain of row biases. */
int hefv_add_part0(hefv_ctx* ctx, uint32_t* rows, int64_t row_stride, const int32_t* slot,
                   const uint32_t* add, int64_t P, void* stream);

/* ---- key switch through an auxiliary basis (K4, second formulation) ----
 * The same result as hefv_keyswitch -- d_j = (sum_i c_i (*) B_ji) mod p_j,
 * fv.py:205-217 -- computed exactly as an integer convolution in the basis of
 * three ~28-bit NTT primes primes32[aux_base .. aux_base+3) and reduced mod
 * p_j: 3k forward + 6k inverse transforms instead of k^2 + 2k.
 * hefv_ks_aux_setup: after hefv_fv_setup; validates the bound
 *   8 k N max(q_j)^2 < a_0 a_1 a_2 and k a_t^2 < 2^62 (k <= 24).
 * hefv_ks_aux_key: switch key (k, k, N) Montgomery device order (as for
 *   hefv_keyswitch) -> kaux (3, 2k, k, N) = NTT_{a_t}(iNTT_j(K_ji)), parts
 *   [body j | mask j]; hefv_ks_aux_key_words gives its size in words.
 * hefv_keyswitch_aux: arguments as hefv_keyswitch, plus
 *   dig_slot: item b's digit rows come from digits + dig_slot[b] * dig_stride
 *     (NULL: b * dig_stride);
 *   galois_elt: if nonzero, the digits are sigma_g(c) of those rows -- the
 *     automorphism of a rotation hop (fv.py:157-173) fused into the load;
 *   scratch of scratch_cts * 9 k N words (ciphertexts are processed in chunks
 *     of scratch_cts). */
int hefv_ks_aux_setup(hefv_ctx* ctx, int32_t aux_base);
int hefv_ks_aux_key(hefv_ctx* ctx, const uint32_t* kbody, const uint32_t* kmask, uint32_t* kaux,
                    void* stream);
int hefv_ks_aux_key_words(hefv_ctx* ctx, int64_t* words);
int hefv_keyswitch_aux(hefv_ctx* ctx, const uint32_t* kaux, const uint32_t* digits,
                       int64_t dig_stride, const int32_t* dig_slot, uint32_t galois_elt,
                       uint32_t* out0, uint32_t* out1, int64_t out_stride,
                       const int32_t* slot, const uint32_t* adA0, const uint32_t* adA1,
                       int64_t adA_stride, const uint32_t* adB0, const uint32_t* adB1,
                       int64_t adB_stride, uint32_t* scratch, int64_t scratch_cts, int64_t B,
                       void* stream);

/* ---- 64-bit RNS key switch (config-4 microbench; _keyswitch_apply,
 * fv.py:205-217, for 50-62-bit primes) --------------------------------------
 * Context: the L 64-bit primes of the context.  kbody/kmask: (L, L, N) =
 * [target j][digit i], device NTT order, Montgomery form (x * 2^64 mod p_j);
 * digits: (B, L, N) coefficient limbs; out: (B, 2, L, N) coefficient domain;
 * scratch: B * L * L * N words. */
int hefv_keyswitch64(hefv_ctx* ctx, const uint64_t* kbody, const uint64_t* kmask,
                     const uint64_t* digits, uint64_t* out, uint64_t* scratch, int64_t B,
                     void* stream);
/* (rows, L, N) -> Montgomery form x * 2^64 mod p_j. */
int hefv_to_montgomery64(hefv_ctx* ctx, const uint64_t* in, uint64_t* out, int64_t rows,
                         void* stream);

/* ---- 64-bit RNS key switch through an aux basis (same limbs as
 * hefv_keyswitch64; fv.py:205-217) ------------------------------------------
 * The context holds the L <= 8 64-bit primes and, as its 32-bit prime set,
 * exactly T aux NTT primes (a_t < 2^62 / L squared-bound, prod a_t > 8 L N
 * max(p)^2); hefv_ks64_aux_setup(ctx, T) validates and tabulates the CRT.
 * hefv_ks64_aux_key: kbody/kmask (L, L, N) [target j][digit i], device NTT
 * order, plain residues -> kaux (T, 2L, L, N) u32; scratch (4 + T) L L N u64.
 * hefv_keyswitch64_aux: digits (B, L, N) coefficient limbs -> out (B, 2, L, N)
 * coefficient domain; scratch B * 3 * L * T * N u32. */
int hefv_ks64_aux_setup(hefv_ctx* ctx, int32_t T);
int hefv_ks64_aux_key(hefv_ctx* ctx, const uint64_t* kbody, const uint64_t* kmask,
                      uint32_t* kaux, uint64_t* scratch, void* stream);
int hefv_keyswitch64_aux(hefv_ctx* ctx, const uint32_t* kaux, const uint64_t* digits,
                         uint64_t* out, uint32_t* scratch, int64_t B, void* stream);

/* ---- object-level surface ---------------------------------
 * What a host without torch needs to run the reference's FvBackend ops
 * (fv.py:254-432) on the device.  Ciphertexts are device buffers of
 * (nparts, k, N) uint32 residues; host buffers use the reference's int64
 * (nparts, k, N) layout (FvCiphertext.parts, fv.py:30-42; serialize.py:80-85).
 * Switch keys are opaque handles.  Plaintext slot vectors are DEVICE
 * (N/2) uint64 arrays of residues mod t (engine.py:138-153 pads them).
 * Temporaries are stream-ordered (cudaMallocAsync on `stream`); unless noted,
 * `out` may alias an input. */
typedef struct hefv_key hefv_key;

/* cudaMalloc / cudaFree of one (nparts, k, N) ciphertext buffer. */
int hefv_ct_alloc(hefv_ctx* ctx, int32_t nparts, uint32_t** out);
int hefv_ct_free(hefv_ctx* ctx, uint32_t* ct);
/* Host int64 (nparts, k, N) <-> device; upload rejects residues outside
 * [0, p_j) (the reference reads them with `% p`, fv.py:30-42). Synchronous. */
int hefv_ct_upload(hefv_ctx* ctx, const int64_t* host, int32_t nparts, uint32_t* ct,
                   void* stream);
int hefv_ct_download(hefv_ctx* ctx, const uint32_t* ct, int32_t nparts, int64_t* host,
                     void* stream);

/* Switch key (fv.py:67-72, _keyswitch_key fv.py:176-202) in the reference's
 * stored form: body/mask (k, k, N) int64 = [target prime j][digit i][natural
 * NTT order], as serialize.read_keyset returns it.  Checked, permuted to
 * device order and Montgomery form on the device, and (when the context has
 * hefv_ks_aux_setup) converted to the aux-basis form.  Synchronous. */
int hefv_key_upload(hefv_ctx* ctx, const int64_t* body, const int64_t* mask, hefv_key** out,
                    void* stream);
/* Handle over device-resident key material already in the device layout
 * (hefv_keygen_digit output; aux form from hefv_ks_aux_key, required when
 * the context uses the aux key switch).  Does not take ownership. */
int hefv_key_wrap(hefv_ctx* ctx, const uint32_t* body, const uint32_t* mask, const uint32_t* aux,
                  hefv_key** out);
int hefv_key_free(hefv_key* key);

/* _encrypt (fv.py:317-335) of B slot vectors (B, N/2): encode, Delta m, then
 * hefv_encrypt with the host-drawn u, e1, e2 (B, N).  out (B, 2, k, N). */
int hefv_encrypt_slots(hefv_ctx* ctx, const uint32_t* pk_ntt, const int8_t* u, const int8_t* e1,
                       const int8_t* e2, const uint64_t* slots, uint32_t* out, int64_t B,
                       void* stream);
/* _decrypt (fv.py:337-353): B ciphertexts of nparts parts -> (B, N/2) slots. */
int hefv_decrypt_slots(hefv_ctx* ctx, const uint32_t* ct, int32_t nparts, const uint32_t* s_ntt,
                       const uint32_t* s2_ntt, uint64_t* slots, int64_t B, void* stream);
/* _add (fv.py:355-357): limb-wise sum of nparts parts. */
int hefv_add(hefv_ctx* ctx, const uint32_t* a, const uint32_t* b, int32_t nparts, uint32_t* out,
             void* stream);
/* _add_plain (fv.py:359-362): c0 + Delta * encode(slots), other parts copied. */
int hefv_add_plain(hefv_ctx* ctx, const uint32_t* ct, int32_t nparts, const uint64_t* slots,
                   uint32_t* out, void* stream);
/* _cmult (fv.py:364-375): every part times centred(encode(slots)). */
int hefv_cmult(hefv_ctx* ctx, const uint32_t* ct, int32_t nparts, const uint64_t* slots,
               uint32_t* out, void* stream);
/* One rotation hop of _rotate (fv.py:417-432): out = (sigma_g(c0), 0) +
 * KS_key(sigma_g(c1)), g = 3^offset mod 2N and `key` the Galois key of that
 * offset.  A rotation by an offset without its own key is the ascending
 * power-of-two hops (fv.py:422-425), one call each. */
int hefv_rotate(hefv_ctx* ctx, const uint32_t* ct, uint32_t galois_elt, const hefv_key* key,
                uint32_t* out, void* stream);
/* _mult + _relinearize (fv.py:377-415): exact BFV tensor of two 2-part
 * ciphertexts (b may equal a) and the relinearisation key switch. */
int hefv_mult(hefv_ctx* ctx, const uint32_t* a, const uint32_t* b, const hefv_key* relin,
              uint32_t* out, void* stream);

/* ---- batched layer rows (the planner; inference.py:261-349) --------------
 * x: (x_cts, 2, k, N) layer input ciphertexts.  R rows, grouped by output
 * ciphertext (row_out ascending); row r: output ciphertext row_out[r] < nout,
 * slot offset row_off[r] (= out_index % s; its piece is rotated by -off),
 * bias row_bias[r] mod t (0 = none; row_bias may be NULL), plaintexts
 * [row_ptr[r], row_ptr[r+1]) -- plaintext p multiplies input ciphertext
 * plain_seg[p] and has entries [plain_ptr[p], plain_ptr[p+1]) of (slot
 * slot_idx[e] < N/2, value slot_val[e] < t).  AllSum has n_iter steps
 * (shift 2^j); Galois keys by rotation offset (key_offsets[i] -> keys[i])
 * must include every power of two below 2^n_iter and every placement hop.
 * The pieces are ADDED into out (nout, 2, k, N).  All plan arrays are host
 * memory; work: device words >= hefv_layer_rows_work_words(...);
 * ks_scratch: ks_cts * 9 k N words (aux key switch; may be NULL otherwise).
 * Same limbs as the reference's per-row loop. */
int hefv_layer_rows_work_words(hefv_ctx* ctx, int32_t x_cts, int64_t R, const int64_t* row_ptr,
                               int64_t tile_rows, int64_t* words);
int hefv_layer_rows(hefv_ctx* ctx, const uint32_t* x, int32_t x_cts, int64_t R,
                    const int32_t* row_out, const int32_t* row_off, const uint64_t* row_bias,
                    const int64_t* row_ptr, const int32_t* plain_seg, const int64_t* plain_ptr,
                    const int32_t* slot_idx, const uint64_t* slot_val, int32_t n_iter,
                    int32_t slot_count, int32_t nkeys, const int32_t* key_offsets,
                    hefv_key* const* keys, uint32_t* out, int32_t nout, int64_t tile_rows,
                    uint32_t* work, int64_t work_words, uint32_t* ks_scratch, int64_t ks_cts,
                    void* stream);

/* ---- key-switch accounting --------------------------------------------------
 * Every hefv_keyswitch / hefv_keyswitch_aux call (direct or from the ops
 * above) is counted; with timing enabled a CUDA event pair brackets it on
 * its stream.  hefv_ks_timing resets; hefv_ks_stats synchronises on the
 * recorded events and returns calls, ciphertexts and the summed ms. */
int hefv_ks_timing(hefv_ctx* ctx, int32_t enable);
int hefv_ks_stats(hefv_ctx* ctx, int64_t* calls, int64_t* cts, double* ms);
/* Cumulative bytes the library itself copied host -> device (layer plans,
 * hefv_ct_upload, hefv_key_upload) and device -> host (hefv_ct_download). */
int hefv_transfer_stats(hefv_ctx* ctx, int64_t* h2d, int64_t* d2h);

/* ---- measurement ---------------------------------------------------------
 * Integer-pipe throughput probe (roofline denominator; not a reference
 * function): kind 0 IMAD, 1 IMAD.HI, 2 IMAD.WIDE, 3 IADD3, 4 Shoup butterfly;
 * executes blocks * 256 * iters * 128 operations. */
int hefv_probe_int(int32_t kind, int32_t blocks, int32_t iters, uint32_t* out, void* stream);
/* tcgen05 int8 check: C (128 x 256 s32) = A (128 x 32ks u8) x B (256 x 32ks u8)^T. */
int hefv_probe_umma(const uint8_t* A, const uint8_t* B, int32_t* C, int32_t ks, void* stream);
/* TMEM load-shape check (development aid): out[t * 4 + r] = register r of thread t. */
int hefv_probe_tmem_shape(int32_t* out, int32_t shape, void* stream);
/* tcgen05 MMA latency / throughput (development aid). */
int hefv_probe_umma_lat(int64_t* out, int32_t reps, int32_t chain, int32_t depth, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HEFV_H */
