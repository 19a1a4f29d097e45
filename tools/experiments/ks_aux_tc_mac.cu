// MEASURED AND REJECTED -- not built into libhefv.so (kept as the record of
// the experiment).
//
// The aux key switch's phase-2 contraction on the int8 tensor cores
// (tcgen05.mma kind::i8, TMEM accumulators): exact -- all aux key-switch
// tests passed bit for bit against the per-prime key switch -- but slower:
// 34.7 us per key switch instead of 20.9 (ksa_bench, B = 1024).  With the
// builders and the epilogue compiled out the bare MMA pipeline alone cost
// ~9 us per key switch, more than the whole integer-pipe contraction (8.1):
// a tcgen05.mma of this size takes ~100 cycles whatever its M x N (64 x 128
// to 128 x 256 measured equal, tools/umma_check.py), and each commit group
// adds ~600; a point needs 3 (K = 96) and its 44 x 7 partial products then
// cost ~14 instructions per output to recombine at 11 of 32 TMEM lanes.
// It was a drop-in for k_ksa_mac in ks_aux.cu (same X / Y layouts; the key
// converted per point into the K-major interleaved u8 operand by
// k_ksa_key8) and needed csrc/umma.cuh.

// ---- phase 2: per-point contraction over digits, on the tensor cores -------
// Y[b][t][jp][point] = (sum_i X[b][t][i][point] K[t][jp][i][point]) 2^-32 mod a_t.
// The sum is exact integer arithmetic (< k a_t^2 < 2^61.1), so it is computed
// on the int8 tensor cores from the bytes of the operands and reduced once:
// with x = sum_u x_u 256^u and k = sum_v k_v 256^v (bytes, u, v < 4),
//   sum_i x k = sum_s C_s 256^s,  C_s = sum_i sum_v k_v[i] x_{s-v}[i]  (s < 7),
// one UMMA per point: D[jp][(b, s)] = A[jp][(i, v)] x B[(b, s)][(i, v)] with
//   A = the key bytes (row jp, K index 4 i + v) -- the key word itself,
//   B = for ciphertext b and shift s, the word (x_s, x_{s-1}, x_{s-2}, x_{s-3})
//       of each digit = byte-reversed x shifted by s - 3 bytes (0 outside),
// u8 x u8 -> s32, every C_s < 2^23 (<= 96 products < 2^16): no overflow.
// The epilogue rebuilds sum_s C_s 256^s in 64 bits (C_4.. C_6 fit one 32-bit
// word because the top bytes are < 19) and Montgomery-reduces it: the same
// canonical Y as any exact evaluation (the reference's: fv.py:205-217 via the
// aux-basis argument above).
//
// M = 64 rows: output jp sits at row 16 (jp / per) + jp % per, per =
// ceil(2k / 4), so after the MMA warp q of the epilogue warpgroup finds it in
// TMEM lane 32 q + jp % per (M = 64 places row r at lane (r % 16) + 32 (r / 16)).
// N = 8 KSA_TC_NB columns (KSA_TC_NB ciphertexts x 8 shifts), K = 32 KS bytes.
//
// CTA = (aux prime t, 32-point tile m, KSA_MAC_CTS ciphertexts); 17 warps:
//   warps 8-15 build B (shared memory, per point) from the bulk-copied digit
//   tiles; warp 16's lane 0 issues the MMAs, commits, and the bulk copies
//   (digit tiles per group of KSA_TC_NB ciphertexts, the key operand per
//   point); warps 0-7 run the epilogue (warp w reads TMEM lane quarter w % 4,
//   half the ciphertexts each).
// Rings: 2 digit stages, KSA_TC_AR key operands, KSA_TC_BR B operands, 4
// accumulators (4 x 128 TMEM columns), all handed over by mbarriers: x / xf
// (digit stage filled / read by every builder warp), a (key operand
// landed), b / bf (B built by every builder warp / read by its MMA), m (MMA
// complete: accumulator full), f (accumulator read by the 8 epilogue warps).

constexpr int KSA_TC_NB = 16;  // ciphertexts per MMA: N = 128 columns
constexpr int KSA_TC_AR = 8;   // key-operand ring (prefetched AR - 2 points ahead)
constexpr int KSA_TC_BR = 4;   // B-operand ring

__host__ __device__ inline int ksa_tc_per(int k) { return (2 * k + 3) / 4; }
__host__ __device__ inline int ksa_tc_ks(int k) { return (4 * k + 31) / 32; }
__host__ __device__ inline uint32_t ksa_tc_abytes(int k) { return 64u * 32u * ksa_tc_ks(k); }

__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_tx(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* mbar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(d),
      "l"(src), "r"(bytes), "r"(m)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* mbar) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

// Montgomery reduction of s < 2^61.2: s 2^-32 mod a, canonical
// ((s + m a) / 2^32 < 2^29.1 + a < 4 a for a > 2^28).
__device__ __forceinline__ uint32_t redc61(uint64_t s, uint32_t a, uint32_t nainv) {
  const uint32_t m = (uint32_t)s * nainv;
  s += (uint64_t)m * a;
  uint32_t v = (uint32_t)(s >> 32);
  v = min(v, v - 2 * a);
  return min(v, v - a);
}

template <int KS>
struct KsaTcSmem {
  static constexpr uint32_t KB = 32 * KS;
  static constexpr uint32_t A_BYTES = 64 * KB;
  static constexpr uint32_t B_BYTES = KSA_TC_NB * 8 * KB;
  static __host__ __device__ constexpr uint32_t x_stride(int k) { return (uint32_t)k * 32 + 4; }
  static __host__ __device__ constexpr size_t bytes(int k) {
    return KSA_TC_AR * (size_t)A_BYTES + KSA_TC_BR * (size_t)B_BYTES +
           2 * (size_t)KSA_TC_NB * x_stride(k) * 4 + 1024;
  }
};

template <int KS>
__global__ void __launch_bounds__(544, 1)
    k_ksa_mac_tc(const uint32_t* __restrict__ X, const uint8_t* __restrict__ kaux8,
                 uint32_t* __restrict__ Y, int64_t B, int k, int log_n, int aux_base,
                 const Prime32Info* __restrict__ info) {
  typedef KsaTcSmem<KS> SM;
  constexpr uint32_t KB = SM::KB, A_BYTES = SM::A_BYTES, B_BYTES = SM::B_BYTES;
  constexpr uint32_t LBO = 128, SBO = 128 * (KB / 16);
  constexpr int NB = KSA_TC_NB;
  extern __shared__ __align__(16) unsigned char smraw[];
  // operands 128-byte aligned (the descriptors need 16); offsets keep the
  // pointers in the shared window (LDS / STS, not generic accesses)
  unsigned char* base = smraw + ((128u - ((uint32_t)__cvta_generic_to_shared(smraw) & 127u)) & 127u);
  unsigned char* As = base;                 // [4][A_BYTES]
  unsigned char* Bs = As + KSA_TC_AR * A_BYTES;  // [2][B_BYTES]
  uint32_t* Xs = reinterpret_cast<uint32_t*>(Bs + KSA_TC_BR * B_BYTES);  // [2][NB][xstride]
  __shared__ __align__(8) uint64_t bar_x[2], bar_xf[2], bar_a[KSA_TC_AR], bar_b[KSA_TC_BR],
      bar_bf[KSA_TC_BR], bar_m[4], bar_f[4];
  __shared__ uint32_t tslot;
  const int n = 1 << log_n;
  const int tiles = n >> 5;
  const int t = blockIdx.x / tiles;
  const int m = blockIdx.x - t * tiles;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t xstride = SM::x_stride(k);
  const uint32_t xbytes = (uint32_t)k * 32 * 4;
  const int64_t bbeg = (int64_t)blockIdx.y * KSA_MAC_CTS;
  const int64_t bend = min(B, bbeg + KSA_MAC_CTS);
  const int ngroups = (int)((bend - bbeg + NB - 1) / NB);
  const int npts = ngroups * 32;  // MMAs of this CTA (u = 32 g + p)
  const size_t xct = (size_t)3 * tiles * k * 32;  // X words per ciphertext
  const uint32_t* xsrc = X + (((size_t)bbeg * 3 + t) * tiles + m) * k * 32;
  const uint8_t* asrc = kaux8 + ((size_t)t * n + (size_t)m * 32) * A_BYTES;
  if (tid == 0) {
    for (int q = 0; q < 2; ++q) {
      mbar_init(&bar_x[q], 1);
      mbar_init(&bar_xf[q], 8);  // the 8 builder warps
    }
    for (int q = 0; q < KSA_TC_BR; ++q) {
      mbar_init(&bar_b[q], 8);
      mbar_init(&bar_bf[q], 1);
    }
    for (int q = 0; q < KSA_TC_AR; ++q) mbar_init(&bar_a[q], 1);
    for (int q = 0; q < 4; ++q) {
      mbar_init(&bar_m[q], 1);
      mbar_init(&bar_f[q], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) tmem_alloc(&tslot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = tslot;
  auto issue_x = [&](int g) {  // digit tiles of group g into stage g % 2
    const int64_t b0 = bbeg + (int64_t)g * NB;
    const int cnt = (int)(bend - b0 < NB ? bend - b0 : NB);
    uint64_t* bar = &bar_x[g & 1];
    mbar_expect_tx(bar, (uint32_t)cnt * xbytes);
    uint32_t* dst = Xs + (size_t)(g & 1) * NB * xstride;
    for (int bl = 0; bl < cnt; ++bl)
      bulk_g2s_tx(dst + (size_t)bl * xstride, xsrc + (size_t)(g * NB + bl) * xct, xbytes, bar);
  };
  auto issue_a = [&](int u) {  // key operand of point u % 32 into slot u % 4
    uint64_t* bar = &bar_a[u % KSA_TC_AR];
    mbar_expect_tx(bar, A_BYTES);
    bulk_g2s_tx(As + (size_t)(u % KSA_TC_AR) * A_BYTES, asrc + (size_t)(u & 31) * A_BYTES, A_BYTES,
                bar);
  };
  if (w == 16) {
    // ---------------- MMA issue + bulk copies (one thread) ----------------
    if (lane == 0) {
      fence_async_smem();
      issue_x(0);
      if (ngroups > 1) issue_x(1);
      for (int u = 0; u < KSA_TC_AR - 2 && u < npts; ++u) issue_a(u);
      const uint32_t idesc = umma_idesc_u8(64, 8 * NB);
      const uint32_t a_sm = (uint32_t)__cvta_generic_to_shared(As);
      const uint32_t b_sm = (uint32_t)__cvta_generic_to_shared(Bs);
      for (int u = 0; u < npts; ++u) {
        const int g = u >> 5;
        mbar_wait(&bar_b[u % KSA_TC_BR], (uint32_t)((u / KSA_TC_BR) & 1));       // B built
        mbar_wait(&bar_a[u % KSA_TC_AR], (uint32_t)((u / KSA_TC_AR) & 1));       // key landed
        if (u >= 4) mbar_wait(&bar_f[u & 3], (uint32_t)(((u - 4) >> 2) & 1));  // acc read
        tmem_fence_after();
        const uint32_t ad = a_sm + (uint32_t)(u % KSA_TC_AR) * A_BYTES;
        const uint32_t bd = b_sm + (uint32_t)(u % KSA_TC_BR) * B_BYTES;
        const uint32_t td = tbase + (uint32_t)(u & 3) * (8 * NB);
#pragma unroll
        for (int q = 0; q < KS; ++q)
          umma_u8(td, umma_smem_desc(ad + 2 * LBO * q, LBO, SBO),
                  umma_smem_desc(bd + 2 * LBO * q, LBO, SBO), idesc, q > 0);
        umma_commit(&bar_m[u & 3]);  // one commit per point: accumulator full, B slot free
        // key operand of point u + AR - 2 into the slot MMA u - 2 read
        if (u + KSA_TC_AR - 2 < npts) {
          if (u >= 2) mbar_wait(&bar_m[(u - 2) & 3], (uint32_t)(((u - 2) >> 2) & 1));
          issue_a(u + KSA_TC_AR - 2);
        }
        // digit stage of group g + 2 once the builders are done with group g
        if ((u & 31) == 31 && g + 2 < ngroups) {
          mbar_wait(&bar_xf[g & 1], (uint32_t)((g >> 1) & 1));
          fence_async_smem();
          issue_x(g + 2);
        }
      }
    }
  } else if (w >= 8) {
    // ---------------- B builders (warps 8-15) ----------------
    const int bt = tid - 256;
    // units (ciphertext bl, 16-byte digit group c, shift s), 256 threads:
    // s = bt & 7 is fixed per thread (a warp's STS.128 fill whole 128-byte
    // rows); precomputed offsets of this thread's UPT units
    constexpr int UNITS = NB * (int)(KB / 16) * 8;
    constexpr int UPT = UNITS / 256;
    static_assert(UNITS % 256 == 0, "unit split");
    const int s_ = bt & 7;
    const bool s7 = s_ == 7;
    const uint32_t sh = 8u * (uint32_t)(6 - (s_ < 7 ? s_ : 6));  // right shift of (r:0) << 24
    uint32_t xoff[UPT], boff[UPT], dmask[UPT];
    int ublj[UPT];
#pragma unroll
    for (int j = 0; j < UPT; ++j) {
      const int rest = (bt >> 3) + 32 * j;
      const int c = rest % (int)(KB / 16), bl = rest / (int)(KB / 16);
      ublj[j] = bl;
      xoff[j] = (uint32_t)bl * xstride + (uint32_t)(4 * c) * 32;
      boff[j] = (uint32_t)bl * SBO + (uint32_t)c * LBO + (uint32_t)s_ * 16;
      uint32_t msk = 0;
      for (int e = 0; e < 4; ++e) msk |= (4 * c + e < k ? 1u : 0u) << e;
      dmask[j] = msk;
    }
    for (int g = 0; g < ngroups; ++g) {
      mbar_wait(&bar_x[g & 1], (uint32_t)((g >> 1) & 1));
      const uint32_t* xs = Xs + (size_t)(g & 1) * NB * xstride;
      const int cnt = (int)(bend - (bbeg + (int64_t)g * NB) < NB ? bend - (bbeg + (int64_t)g * NB) : NB);
      for (int p = 0; p < 32; ++p) {
        const int u = g * 32 + p;
        // B slot u % 4 was last read by MMA u - 4 (its commit is bar_m[u & 3])
        if (u >= 4) mbar_wait(&bar_m[u & 3], (uint32_t)(((u - 4) >> 2) & 1));
        unsigned char* bsl = Bs + (size_t)(u % KSA_TC_BR) * B_BYTES;
#ifndef KSA_TC_NOBUILD
#pragma unroll
        for (int j = 0; j < UPT; ++j) {
          uint32_t wv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t xw = ((dmask[j] >> e) & 1u) && ublj[j] < cnt ? xs[xoff[j] + e * 32 + p] : 0u;
            const uint32_t r = __byte_perm(xw, 0u, 0x0123);  // byte-reversed digit
            // (x_s, x_{s-1}, x_{s-2}, x_{s-3}) = ((r:0) << 24) >> 8 (6 - s), 0 for s = 7
            wv[e] = s7 ? 0u : (sh < 32 ? __funnelshift_r(r << 24, r >> 8, sh) : (r >> (sh - 24)));
          }
          *reinterpret_cast<uint4*>(bsl + boff[j]) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
#endif
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive1(&bar_b[u % KSA_TC_BR]);  // this warp's share is built
      }
      __syncwarp();
      if (lane == 0) mbar_arrive1(&bar_xf[g & 1]);  // done reading this digit stage
    }
  } else {
    // ---------------- epilogue: warp w reads TMEM lane quarter w % 4 ----------
    const int q = w & 3;
    const int half = w >> 2;  // ciphertexts [half NB/2, (half + 1) NB/2) of each MMA
    const int per = ksa_tc_per(k);
    const int jp = q * per + lane;
    const bool active = lane < per && jp < 2 * k;
    const uint32_t a = info[aux_base + t].p;
    uint32_t nainv;
    {
      uint32_t inv = a;
#pragma unroll
      for (int it = 0; it < 5; ++it) inv *= 2u - a * inv;
      nainv = 0u - inv;
    }
    uint32_t* yrow = Y + ((size_t)t * 2 * k + (active ? jp : 0)) * (size_t)n + (size_t)m * 32;
    const size_t ystride = (size_t)3 * 2 * k * n;  // per ciphertext
    constexpr int HB = NB / 2;                      // this warp's ciphertexts per MMA
    for (int u = 0; u < npts; ++u) {
      const int g = u >> 5, p = u & 31;
      const int64_t b0 = bbeg + (int64_t)g * NB + half * HB;
      const int nv = (int)(bend - b0 < HB ? (bend - b0 < 0 ? 0 : bend - b0) : HB);
      mbar_wait(&bar_m[u & 3], (uint32_t)((u >> 2) & 1));
      tmem_fence_after();
      const uint32_t tacc = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(u & 3) * (8 * NB) +
                            (uint32_t)(half * HB * 8);
      uint32_t v[HB][8];
#ifndef KSA_TC_NOEPI
#pragma unroll
      for (int e = 0; e < HB; ++e) tmem_ld8(tacc + 8 * e, v[e]);
      tmem_wait_ld();
#else
      for (int e = 0; e < HB; ++e) for (int z = 0; z < 8; ++z) v[e][z] = 0;
#endif
      tmem_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive1(&bar_f[u & 3]);  // accumulator read: hand it back
#ifdef KSA_TC_NOEPI
      if (false) {
#else
      if (active) {
#endif
        uint32_t* yp = yrow + (size_t)b0 * ystride + p;
#pragma unroll
        for (int e = 0; e < HB; ++e) {
          if (e < nv) {
            const uint64_t P = (uint64_t)v[e][0] + ((uint64_t)v[e][1] << 8) +
                               ((uint64_t)v[e][2] << 16) + ((uint64_t)v[e][3] << 24);
            const uint32_t Q = v[e][4] + (v[e][5] << 8) + (v[e][6] << 16);
            yp[e * ystride] = redc61(P + ((uint64_t)Q << 32), a, nainv);
          }
        }
      }
    }
  }
  tmem_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, 512);
}

// Switch key, tiled aux form (3, 2k, k, N) words -> the tensor-core operand
// form: per (aux prime t, point) a 64-row x 32 KS-byte K-major operand in
// the interleaved canonical layout, row of jp as in k_ksa_mac_tc, the key
// word K[t][jp][i] at bytes 4 i .. 4 i + 3 (zero elsewhere).
__global__ void k_ksa_key8(const uint32_t* __restrict__ kaux, uint32_t* __restrict__ kaux8, int k,
                           int log_n) {
  const int n = 1 << log_n, tiles = n >> 5;
  const int ks = ksa_tc_ks(k), per = ksa_tc_per(k);
  const uint32_t abytes = ksa_tc_abytes(k), sbo = 128u * (2 * ks);
  const int64_t total = (int64_t)3 * n * 2 * k;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int jp = (int)(g % (2 * k));
    const int64_t tp = g / (2 * k);
    const int point = (int)(tp % n);
    const int t = (int)(tp / n);
    const int mt = point >> 5, l = point & 31;
    const int r = 16 * (jp / per) + jp % per;
    const uint32_t* src = kaux + (((size_t)t * 2 * k + jp) * tiles + mt) * k * 32 + l;
    unsigned char* dst = reinterpret_cast<unsigned char*>(kaux8) + ((size_t)t * n + point) * abytes +
                         (size_t)(r / 8) * sbo + (size_t)(r % 8) * 16;
    for (int i = 0; i < k; ++i)
      *reinterpret_cast<uint32_t*>(dst + (size_t)((4 * i) / 16) * 128 + (4 * i) % 16) =
          src[(size_t)i * 32];
  }
}

