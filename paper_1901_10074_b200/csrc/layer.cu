// Batched layer rows: the device side of the layer planner, in C++.
//
// The reference evaluates a compiled layer one weight row at a time
// (inference.py:277-338): segment cmults summed, AllSum over s slots, bias,
// e0 mask, placement rotation by -off, and an add into out[off // s].  Rows
// are independent until that final modular sum, so hefv_layer_rows runs a
// tile of T rows per launch sequence (see planner.py for the argument that
// the limbs equal the serial schedule's):
//   1. the tile's sparse plaintexts encoded and transformed on the device,
//      one NTT-domain MAC launch for all segment products;
//   2. AllSum step j: one batched rotation hop (automorphism + key switch
//      under the shared Galois key, running sum fused into the epilogue);
//   3. biases (batched add_plain), the e0 mask (batched ct x pt);
//   4. placement: hop h for every row whose rotation contains it, custom
//      keys first, then powers of two ascending (fv.py:422-425);
//   5. per-output-ciphertext sums of the pieces.
// The host part is only bookkeeping: the plan (CSR plaintexts, per-tile hop
// groups and output segments) is built once per call in a pinned staging
// buffer (a per-context pool: a buffer is reused once its copy is done) and
// copied to the device in one transfer.
#include <algorithm>
#include <cstring>
#include <map>
#include <vector>

#include "../../include/hefv.h"
#include "internal.h"

namespace hefv {

static uint32_t galois_of(int64_t offset, int n) {
  // 3^offset mod 2N (ring.galois_element; fv.py:427)
  const uint64_t m = 2ull * (uint64_t)n;
  uint64_t r = 1, b = 3 % m, e = (uint64_t)offset;
  while (e) {
    if (e & 1) r = r * b % m;
    b = b * b % m;
    e >>= 1;
  }
  return (uint32_t)r;
}

// One Galois hop of B ciphertexts (planner.rotation_keyswitch):
// out[out_slot b] = KS(sigma_g(c1)) + (sigma_g(c0), 0) + adB[out_slot b].
static int rotation_hop(hefv_ctx* c, const hefv_key* key, uint32_t* src, int64_t src_stride,
                        const int32_t* slot, uint32_t g, int64_t B, uint32_t* out0,
                        uint32_t* out1, int64_t out_stride, const int32_t* out_slot,
                        const uint32_t* adB0, const uint32_t* adB1, int64_t adB_stride,
                        uint32_t* scratch, uint32_t* ks_scratch, int64_t ks_cts,
                        cudaStream_t st) {
  const int64_t stack = (int64_t)c->k * c->n;
  if (key->aux) {
    if (int r = hefv_automorph(c, src, src_stride, slot, scratch, 1, g, B, st)) return r;
    return hefv_keyswitch_aux(c, key->aux, src + stack, src_stride, slot, g, out0, out1,
                              out_stride, out_slot, scratch, nullptr, stack, adB0, adB1,
                              adB_stride, ks_scratch, ks_cts, B, st);
  }
  if (int r = hefv_automorph(c, src, src_stride, slot, scratch, 2, g, B, st)) return r;
  return hefv_keyswitch(c, key->body, key->mask, scratch + stack, 2 * stack, out0, out1,
                        out_stride, out_slot, scratch, nullptr, 2 * stack, adB0, adB1,
                        adB_stride, B, st);
}

// Host plan of one tile: offsets (bytes) into the staged plan buffer.
struct TilePlan {
  int64_t r0 = 0, B = 0, P = 0, e_lo = 0, g_lo = 0;
  size_t ptr = 0, rp = 0;                 // int32 (P+1), int32 (B+1)
  int64_t nb = 0;
  size_t bslot = 0, bptr = 0, bidx = 0, bval = 0;  // biases
  std::vector<std::pair<int64_t, std::pair<size_t, int64_t>>> hops;  // (offset, (slots, count))
  int32_t M = 0;
  size_t seg = 0, seg_out = 0;
};

struct Stage {
  std::vector<unsigned char> bytes;
  template <class T>
  size_t put(const T* src, size_t count) {
    size_t off = (bytes.size() + 15) & ~size_t(15);
    bytes.resize(off + std::max<size_t>(count, 1) * sizeof(T));
    if (count) std::memcpy(bytes.data() + off, src, count * sizeof(T));
    return off;
  }
};

// plaintext slots of the largest tile (at least T: the bias plaintexts reuse them)
static int64_t tile_plain_max(const int64_t* row_ptr, int64_t R, int64_t T) {
  int64_t pmax = T;
  for (int64_t r0 = 0; r0 < R; r0 += T) {
    const int64_t B = std::min(T, R - r0);
    pmax = std::max(pmax, row_ptr[r0 + B] - row_ptr[r0]);
  }
  return pmax;
}

}  // namespace hefv

using namespace hefv;

extern "C" {

int hefv_layer_rows_work_words(hefv_ctx* c, int32_t x_cts, int64_t R, const int64_t* row_ptr,
                               int64_t tile_rows, int64_t* words) {
  if (!c || !c->fv_ready) return fail("hefv_layer_rows_work_words: context without FV setup");
  if (!words || !row_ptr) return fail("hefv_layer_rows_work_words: null pointer");
  if (tile_rows < 1) return fail("hefv_layer_rows_work_words: tile_rows must be >= 1");
  const int64_t stack = (int64_t)c->k * c->n;
  const int64_t T = std::min<int64_t>(tile_rows, std::max<int64_t>(R, 1));
  const int64_t pmax = tile_plain_max(row_ptr, R, T);
  *words = (int64_t)x_cts * 2 * stack      // NTT(x), Montgomery
           + T * 4 * stack                 // tile accumulators + hop scratch
           + pmax * (stack + 2 * c->n)     // plaintext polys (u64) + their NTTs
           + stack;                        // NTT of centred(encode(e0))
  return 0;
}

int hefv_layer_rows(hefv_ctx* c, const uint32_t* x, int32_t x_cts, int64_t R,
                    const int32_t* row_out, const int32_t* row_off, const uint64_t* row_bias,
                    const int64_t* row_ptr, const int32_t* plain_seg, const int64_t* plain_ptr,
                    const int32_t* slot_idx, const uint64_t* slot_val, int32_t n_iter,
                    int32_t slot_count, int32_t nkeys, const int32_t* key_offsets,
                    hefv_key* const* keys, uint32_t* out, int32_t nout, int64_t tile_rows,
                    uint32_t* work, int64_t work_words, uint32_t* ks_scratch, int64_t ks_cts,
                    void* stream) {
  if (!c || !c->fv_ready) return fail("hefv_layer_rows: context without FV setup");
  if (R <= 0) return 0;
  if (!x || x_cts < 1 || !row_out || !row_off || !row_ptr || !plain_seg || !plain_ptr || !out ||
      !work)
    return fail("hefv_layer_rows: null argument");
  if (tile_rows < 1) return fail("hefv_layer_rows: tile_rows must be >= 1");
  if (c->ksa_ready && (!ks_scratch || ks_cts < 1))
    return fail("hefv_layer_rows: the aux-basis key switch needs a workspace");
  cudaStream_t st = as_stream(stream);
  const int n = c->n;
  const int64_t stack = (int64_t)c->k * n;
  const int64_t ct_words = 2 * stack;
  const int64_t T = std::min<int64_t>(tile_rows, R);

  // ---- keys by rotation offset
  std::map<int64_t, const hefv_key*> kmap;
  for (int i = 0; i < nkeys; ++i) {
    if (!keys[i] || keys[i]->ctx != c) return fail("hefv_layer_rows: key of another context");
    kmap[key_offsets[i]] = keys[i];
  }
  for (int j = 0; j < n_iter; ++j)
    if (!kmap.count((int64_t)1 << j))
      return fail("hefv_layer_rows: missing the power-of-two Galois key " +
                  std::to_string(1 << j));

  // ---- validate the plan
  const int64_t P_all = row_ptr[R] - row_ptr[0];
  if (row_ptr[0] != 0 || P_all < 0) return fail("hefv_layer_rows: bad row_ptr");
  const int64_t E_all = plain_ptr[P_all];
  if (plain_ptr[0] != 0 || E_all < 0) return fail("hefv_layer_rows: bad plain_ptr");
  for (int64_t p = 0; p < P_all; ++p)
    if (plain_seg[p] < 0 || plain_seg[p] >= x_cts)
      return fail("hefv_layer_rows: plaintext segment outside the input ciphertexts");
  for (int64_t p = 0; p < P_all; ++p)
    if (plain_ptr[p + 1] < plain_ptr[p]) return fail("hefv_layer_rows: plain_ptr not monotone");
  for (int64_t e = 0; e < E_all; ++e)
    if (slot_idx[e] < 0 || slot_idx[e] >= n / 2 || slot_val[e] >= c->t)
      return fail("hefv_layer_rows: plaintext entry outside [0, N/2) x [0, t)");
  for (int64_t r = 0; r < R; ++r) {
    if (row_out[r] < 0 || row_out[r] >= nout) return fail("hefv_layer_rows: bad row_out");
    if (row_bias && row_bias[r] >= c->t) return fail("hefv_layer_rows: bias not reduced mod t");
    if (r && row_out[r] < row_out[r - 1])
      return fail("hefv_layer_rows: rows must be grouped by output ciphertext (ascending)");
    if (row_ptr[r + 1] < row_ptr[r]) return fail("hefv_layer_rows: row_ptr not monotone");
  }
  int64_t need = 0;
  if (int r = hefv_layer_rows_work_words(c, x_cts, R, row_ptr, T, &need)) return r;
  if (work_words < need)
    return fail("hefv_layer_rows: workspace too small (" + std::to_string(need) + " words needed)");

  // ---- host plan, staged in one buffer
  Stage sg;
  const size_t o_slot = sg.put(slot_idx, (size_t)E_all);
  const size_t o_val = sg.put(slot_val, (size_t)E_all);
  const size_t o_seg = sg.put(plain_seg, (size_t)P_all);
  // the one-hot e0 as a sparse plaintext: slot 0 = 1
  const int32_t e0ptr[2] = {0, 1}, e0idx[1] = {0};
  const uint64_t e0val[1] = {1};
  const size_t o_e0ptr = sg.put(e0ptr, 2), o_e0idx = sg.put(e0idx, 1), o_e0val = sg.put(e0val, 1);
  std::vector<TilePlan> tiles;
  for (int64_t r0 = 0; r0 < R; r0 += T) {
    TilePlan tp;
    tp.r0 = r0;
    tp.B = std::min(T, R - r0);
    tp.g_lo = row_ptr[r0];
    tp.P = row_ptr[r0 + tp.B] - tp.g_lo;
    tp.e_lo = plain_ptr[tp.g_lo];
    std::vector<int32_t> ptr(tp.P + 1), rp(tp.B + 1);
    for (int64_t p = 0; p <= tp.P; ++p) ptr[p] = (int32_t)(plain_ptr[tp.g_lo + p] - tp.e_lo);
    for (int64_t b = 0; b <= tp.B; ++b) rp[b] = (int32_t)(row_ptr[r0 + b] - tp.g_lo);
    tp.ptr = sg.put(ptr.data(), ptr.size());
    tp.rp = sg.put(rp.data(), rp.size());
    // biases (slot 0 of part 0, fv.py:355-362)
    std::vector<int32_t> bslot, bptr(1, 0), bidx;
    std::vector<uint64_t> bval;
    for (int64_t b = 0; b < tp.B; ++b) {
      const uint64_t v = row_bias ? row_bias[r0 + b] : 0;
      if (!v) continue;
      bslot.push_back((int32_t)b);
      bidx.push_back(0);
      bval.push_back(v);
      bptr.push_back((int32_t)bslot.size());
    }
    tp.nb = (int64_t)bslot.size();
    tp.bslot = sg.put(bslot.data(), bslot.size());
    tp.bptr = sg.put(bptr.data(), bptr.size());
    tp.bidx = sg.put(bidx.data(), bidx.size());
    tp.bval = sg.put(bval.data(), bval.size());
    // placement hops: rotation by -off decomposed as the backend does
    // (one hop with a dedicated key, else ascending powers of two)
    std::map<int64_t, std::vector<int32_t>> groups;
    for (int64_t b = 0; b < tp.B; ++b) {
      const int64_t off = row_off[r0 + b];
      if (!off) continue;
      const int64_t rot = ((-off) % slot_count + slot_count) % slot_count;
      if (!rot) continue;
      if (kmap.count(rot)) {
        groups[rot].push_back((int32_t)b);
      } else {
        for (int bit = 0; (rot >> bit) != 0; ++bit)
          if ((rot >> bit) & 1) groups[(int64_t)1 << bit].push_back((int32_t)b);
      }
    }
    std::vector<int64_t> order;
    for (auto& kv : groups)
      if (kv.first & (kv.first - 1)) order.push_back(kv.first);  // custom keys first
    for (auto& kv : groups)
      if (!(kv.first & (kv.first - 1))) order.push_back(kv.first);
    for (int64_t h : order) {
      if (!kmap.count(h)) return fail("hefv_layer_rows: no Galois key for hop " + std::to_string(h));
      auto& v = groups[h];
      tp.hops.push_back({h, {sg.put(v.data(), v.size()), (int64_t)v.size()}});
    }
    // output segments of the tile (rows grouped by output ciphertext)
    std::vector<int32_t> seg(1, 0), seg_out;
    seg_out.push_back(row_out[r0]);
    for (int64_t b = 1; b < tp.B; ++b)
      if (row_out[r0 + b] != row_out[r0 + b - 1]) {
        seg.push_back((int32_t)b);
        seg_out.push_back(row_out[r0 + b]);
      }
    seg.push_back((int32_t)tp.B);
    tp.M = (int32_t)seg_out.size();
    tp.seg = sg.put(seg.data(), seg.size());
    tp.seg_out = sg.put(seg_out.data(), seg_out.size());
    tiles.push_back(std::move(tp));
  }

  // ---- one pinned transfer of the plan
  const size_t plan_bytes = sg.bytes.size();
  // a pinned buffer whose last copy has completed (or a new one)
  hefv_ctx::Stage* stage = nullptr;
  for (auto& cand : c->stages)
    if (cudaEventQuery(cand.done) == cudaSuccess && (!stage || cand.bytes > stage->bytes)) stage = &cand;
  if (!stage) {
    c->stages.emplace_back();
    stage = &c->stages.back();
    HEFV_CUDA(cudaEventCreateWithFlags(&stage->done, cudaEventDisableTiming));
  }
  if (stage->bytes < plan_bytes) {
    if (stage->host) cudaFreeHost(stage->host);
    stage->host = nullptr;
    stage->bytes = 0;
    HEFV_CUDA(cudaMallocHost(&stage->host, plan_bytes));
    stage->bytes = plan_bytes;
  }
  std::memcpy(stage->host, sg.bytes.data(), plan_bytes);
  unsigned char* d_plan = nullptr;
  HEFV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_plan), plan_bytes, st));
  struct PlanFree {
    void* p;
    cudaStream_t st;
    ~PlanFree() { cudaFreeAsync(p, st); }
  } plan_free{d_plan, st};
  HEFV_CUDA(cudaMemcpyAsync(d_plan, stage->host, plan_bytes, cudaMemcpyHostToDevice, st));
  c->h2d_bytes += (int64_t)plan_bytes;
  HEFV_CUDA(cudaEventRecord(stage->done, st));
  auto P32 = [&](size_t off) { return reinterpret_cast<int32_t*>(d_plan + off); };
  auto P64 = [&](size_t off) { return reinterpret_cast<uint64_t*>(d_plan + off); };

  // ---- workspace
  uint32_t* x_ntt = work;
  uint32_t* acc = x_ntt + (int64_t)x_cts * ct_words;
  uint32_t* scr = acc + T * ct_words;
  const int64_t pmax = tile_plain_max(row_ptr, R, T);
  uint64_t* polys = reinterpret_cast<uint64_t*>(scr + T * ct_words);
  uint32_t* m_ntt = reinterpret_cast<uint32_t*>(polys + pmax * n);
  uint32_t* e0 = m_ntt + pmax * stack;

  // NTT (device order, Montgomery form) of the layer inputs, once
  if (int r = hefv_ntt_fwd32(c, x, x_ntt, 2 * (int64_t)x_cts, c->k, 0, 0, st)) return r;
  if (int r = hefv_to_montgomery(c, x_ntt, x_ntt, 2 * (int64_t)x_cts, st)) return r;
  // e0 = NTT(centred(encode(one-hot slot 0))), Montgomery form (inference.py:287, 327)
  if (int r = hefv_encode_sparse(c, P32(o_e0ptr), P32(o_e0idx), P64(o_e0val), polys, 1, st))
    return r;
  if (int r = hefv_plain_to_rns(c, polys, e0, 1, 1, 1, 1, st)) return r;

  for (const TilePlan& tp : tiles) {
    const int64_t B = tp.B;
    uint32_t* a0 = acc;
    uint32_t* a1 = acc + stack;
    // ---- 1. segment products
    if (tp.P) {
      if (int r = hefv_encode_sparse(c, P32(tp.ptr), P32(o_slot) + tp.e_lo, P64(o_val) + tp.e_lo,
                                     polys, tp.P, st))
        return r;
      // plain (non-Montgomery) NTTs: the inputs carry the Montgomery factor
      if (int r = hefv_plain_to_rns(c, polys, m_ntt, tp.P, 1, 1, 0, st)) return r;
      if (int r = hefv_rows_mac(c, x_ntt, m_ntt, P32(tp.rp), P32(o_seg) + tp.g_lo, acc, B, st))
        return r;
    } else {
      HEFV_CUDA(cudaMemsetAsync(acc, 0, (size_t)B * ct_words * 4, st));
    }
    // ---- 2. AllSum over s slots: x <- x + rot(x, 2^j)
    for (int j = 0; j < n_iter; ++j) {
      const int64_t shift = (int64_t)1 << j;
      if (int r = rotation_hop(c, kmap[shift], a0, ct_words, nullptr, galois_of(shift, n), B, a0,
                               a1, ct_words, nullptr, a0, a1, ct_words, scr, ks_scratch, ks_cts,
                               st))
        return r;
    }
    // ---- 3. biases, then the e0 mask
    if (tp.nb) {
      if (int r = hefv_encode_sparse(c, P32(tp.bptr), P32(tp.bidx), P64(tp.bval), polys, tp.nb, st))
        return r;
      if (int r = hefv_plain_to_rns(c, polys, m_ntt, tp.nb, 0, 0, 0, st)) return r;
      if (int r = hefv_add_part0(c, a0, ct_words, P32(tp.bslot), m_ntt, tp.nb, st)) return r;
    }
    if (int r = hefv_mul_plain(c, a0, e0, a0, B, 2, 1, st)) return r;
    // ---- 4. placement rotations by -off
    for (const auto& h : tp.hops) {
      const int32_t* d_slot = P32(h.second.first);
      if (int r = rotation_hop(c, kmap[h.first], a0, ct_words, d_slot, galois_of(h.first, n),
                               h.second.second, a0, a1, ct_words, d_slot, nullptr, nullptr, 0, scr,
                               ks_scratch, ks_cts, st))
        return r;
    }
    // ---- 5. pieces summed into their output ciphertexts
    if (int r = hefv_accumulate_rows(c, a0, P32(tp.seg), P32(tp.seg_out), out, tp.M, 1, st))
      return r;
  }
  return 0;
}

}  // extern "C"
