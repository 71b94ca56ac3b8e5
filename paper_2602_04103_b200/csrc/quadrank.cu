// quadrank.cu — QuadRank16 (sigma = 4, 2-bit DNA) on sm_100a: builder, rank(q,c), rank_4(q).
//
// Layout (§4; Listing 1; R5-R7): line j is
// 8 u64 words = two halves h of 4 words; half h, pair t holds line chars 128h+64t..+63 as
//   word 4h+2t   = NOT(low bits of those 64 chars)    word 4h+2t+1 = NOT(high bits)
// Data char k (global char 224 j + k) is line char 32 + k.  Line chars 0..31 (the low 32
// bits of words 0 and 1) hold the four u16 deltas at u16 slots c + (c & 2):
//   word0 = b_A | b_C << 16 | NOT(low bits of data chars 0..31) << 32
//   word1 = b_G | b_T << 16 | NOT(high bits of data chars 0..31) << 32
// b_{j,c} = rank(224 j + 96, c) - 2^13 s_{j>>8, c}; s_{i,c} = floor(rank(256 i 224, c)/2^13).
// Line j's data chars are exactly text words [7j, 7j+7) (224 = 7 * 32).
//
// Query (Listing 1): j = q / 224, p = 32 + q - 224 j in [32, 256); the anchor is line char
// 128, so p < 128 counts line chars [p,128) of half 0 (sector 0, which also holds the deltas)
// and subtracts; p >= 128 counts [128, p) of half 1 (sector 1) and adds.  Char k matches c
// iff bit k of (w_low ^ cl) & (w_high ^ ch), cl = -(c & 1), ch = -(c >> 1).
#include <cub/device/device_scan.cuh>

#include "qr_common.cuh"
#include "sched.cuh"

namespace qr {

// ------------------------------------------------------------------ build

__device__ __forceinline__ uint32_t sym_counts_word(uint64_t w, uint32_t cnt[4]) {
  const uint64_t M = 0x5555555555555555ull;
  uint64_t lo = w & M, hi = (w >> 1) & M;
  uint32_t c3 = __popcll(lo & hi), l1 = __popcll(lo), h1 = __popcll(hi);
  cnt[3] += c3;
  cnt[1] += l1 - c3;
  cnt[2] += h1 - c3;
  cnt[0] += 32 - l1 - h1 + c3;
  return 0;
}

// per line: counts over data chars [0,96) (c96, u8 x4 packed in a u32) and totals (SoA u64).
__global__ void k_qd_count(const uint64_t* __restrict__ text, uint64_t L, uint32_t* __restrict__ c96,
                           uint64_t* __restrict__ tot) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t* t = text + 7 * j;
    uint32_t a[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 3; ++k) sym_counts_word(t[k], a);
    c96[j] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
#pragma unroll
    for (int k = 3; k < 7; ++k) sym_counts_word(t[k], a);
#pragma unroll
    for (int c = 0; c < 4; ++c) tot[(uint64_t)c * L + j] = a[c];
  }
}

// compact the bits at even positions of x into 32 bits
__device__ __forceinline__ uint64_t even_bits(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return x;
}

__global__ void k_qd_write(const uint64_t* __restrict__ text, uint64_t L, const uint32_t* __restrict__ c96,
                           const uint64_t* __restrict__ R, uint4* __restrict__ lines, uint32_t* __restrict__ super) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t jsb = (j >> QD_SB_LOG) << QD_SB_LOG;
    const uint32_t c96p = c96[j];
    uint32_t b[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint64_t sb = R[(uint64_t)c * L + jsb] >> QD_SHIFT;
      if (j == jsb) super[4 * (j >> QD_SB_LOG) + c] = (uint32_t)sb;
      b[c] = (uint32_t)(R[(uint64_t)c * L + j] + ((c96p >> (8 * c)) & 0xffu) - (sb << QD_SHIFT));
    }
    const uint64_t* t = text + 7 * j;
    uint64_t lo[7], hi[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      uint64_t w = t[k];
      lo[k] = even_bits(w);
      hi[k] = even_bits(w >> 1);
    }
    uint64_t w0 = (uint64_t)(b[0] | (b[1] << 16)) | ((~lo[0]) << 32);
    uint64_t w1 = (uint64_t)(b[2] | (b[3] << 16)) | ((~hi[0]) << 32);
    uint64_t w2 = ~(lo[1] | (lo[2] << 32)), w3 = ~(hi[1] | (hi[2] << 32));
    uint64_t w4 = ~(lo[3] | (lo[4] << 32)), w5 = ~(hi[3] | (hi[4] << 32));
    uint64_t w6 = ~(lo[5] | (lo[6] << 32)), w7 = ~(hi[5] | (hi[6] << 32));
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(lines + 4 * j);
    dst[0] = make_ulonglong2(w0, w1);
    dst[1] = make_ulonglong2(w2, w3);
    dst[2] = make_ulonglong2(w4, w5);
    dst[3] = make_ulonglong2(w6, w7);
  }
}

__global__ void k_mask_tail_chars(uint64_t* words, uint64_t n) {
  uint64_t r = n & 31;
  if (r) words[n >> 5] &= (1ull << (2 * r)) - 1ull;
}

qr_status quadrank_build_device(const uint64_t* d_text, uint64_t n, int device, cudaStream_t st, qr_index** out) {
  // d_text: device copy owned by the caller, >= 7 L words, zero padded beyond n chars.
  qr_index* h = nullptr;
  qr_status rs = alloc_index(4, n, device, &h);
  if (rs != QR_OK) return rs;
  const uint64_t L = h->n_lines;
  uint32_t* c96 = nullptr;
  uint64_t *tot = nullptr, *R = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  auto bail = [&](cudaError_t err, const char* what) {
    cudaFreeAsync(c96, st); cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(tmp, st);
    qr_free(h);
    return cuda_fail(err, what);
  };
  k_mask_tail_chars<<<1, 1, 0, st>>>(const_cast<uint64_t*>(d_text), n);
  if ((e = cudaMallocAsync((void**)&c96, L * sizeof(uint32_t), st))) return bail(e, "alloc c96");
  if ((e = cudaMallocAsync((void**)&tot, 4 * L * sizeof(uint64_t), st))) return bail(e, "alloc tot");
  if ((e = cudaMallocAsync((void**)&R, 4 * L * sizeof(uint64_t), st))) return bail(e, "alloc R");
  unsigned g = grid_stride_blocks(L, 256, h->sm_count, 16);
  k_qd_count<<<g, 256, 0, st>>>(d_text, L, c96, tot);
  if ((e = cudaGetLastError())) return bail(e, "k_qd_count");
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, tot, R, (int64_t)L, st))) return bail(e, "scan size");
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st))) return bail(e, "alloc scan tmp");
  for (int c = 0; c < 4; ++c)
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, tot + (uint64_t)c * L, R + (uint64_t)c * L, (int64_t)L, st)))
      return bail(e, "scan");
  k_qd_write<<<g, 256, 0, st>>>(d_text, L, c96, R, h->lines, h->super);
  if ((e = cudaGetLastError())) return bail(e, "k_qd_write");
  cudaFreeAsync(c96, st); cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(tmp, st);
  if ((rs = build_super_pack(h, st)) != QR_OK) { qr_free(h); return rs; }
  *out = h;
  return QR_OK;
}

// ------------------------------------------------------------------ queries

template <bool SMALLQ>
__device__ __forceinline__ uint64_t qd_line_of(uint64_t q) {
  if (SMALLQ) return (uint64_t)((uint32_t)(q >> 5) / 7u);   // floor(floor(q/32)/7) = floor(q/224), q < 2^37
  return q / QD_B;
}

// masked matching-char count of one half (two plane pairs) for symbol c.
// x = p (left: count [p,128), inv = ~0) or p - 128 (right: count [0, x), inv = 0).
__device__ __forceinline__ uint32_t qd_count(const uint64_t w[4], uint32_t c, int x, uint64_t inv) {
  const uint64_t cl = 0ull - (uint64_t)(c & 1u), ch = 0ull - (uint64_t)(c >> 1);
  uint32_t cnt = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t) cnt += __popcll((w[2 * t] ^ cl) & (w[2 * t + 1] ^ ch) & (prefix_mask(x, t) ^ inv));
  return cnt;
}

template <int K, bool SMALLQ>
__device__ __forceinline__ void qd_locate(const uint64_t (&qq)[K], uint64_t last_line, uint64_t (&jj)[K],
                                          uint32_t (&pp)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uint64_t j = qd_line_of<SMALLQ>(qq[k]);
    j = j > last_line ? last_line : j;                   // q > n: memory-safe clamp
    uint64_t p = 32 + qq[k] - j * QD_B;
    pp[k] = p > 255 ? 255u : (uint32_t)p;
    jj[k] = j;
  }
}

// next group's query positions (and symbols), loaded while the current gathers are in flight
template <int K, bool WITH_C>
__device__ __forceinline__ void qd_load_group(const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                              uint64_t i0, uint64_t nthr, uint64_t m, uint64_t (&qn)[K],
                                              uint32_t (&cn)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uint64_t idx = i0 + (uint64_t)k * nthr;
    qn[k] = idx < m ? ld_stream_u64(q + idx) : 0;
    if (WITH_C) cn[k] = idx < m ? ld_stream_u8(cs + idx) & 3u : 0u;
  }
}

// Same structure as k_bi_rank (K gathers in flight per thread, next group's (q, c) prefetched).
template <int K, bool SMALLQ>
__global__ void __launch_bounds__(256) k_qd_rank(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                 const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                                 uint64_t* __restrict__ out, uint64_t m, uint64_t last_line) {
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t qn[K];
  uint32_t cn[K];
  qd_load_group<K, true>(q, cs, i0, nthr, m, qn, cn);
  for (; i0 < m; i0 += nthr * K) {
    uint64_t qq[K], jj[K];
    uint32_t pp[K], cc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { qq[k] = qn[k]; cc[k] = cn[k]; }
    qd_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t a[K][4], b[K][4];
    uint32_t s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint4* ln = lines + 4 * jj[k];
      ld_sector_na(ln, a[k][0], a[k][1], a[k][2], a[k][3]);
      b[k][0] = b[k][1] = b[k][2] = b[k][3] = 0;
      if (pp[k] >= 128) ld_sector_na(ln + 2, b[k][0], b[k][1], b[k][2], b[k][3]);
      s[k] = __ldg(super + 4 * (jj[k] >> QD_SB_LOG) + cc[k]);
    }
    qd_load_group<K, true>(q, cs, i0 + nthr * K, nthr, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint64_t idx = i0 + (uint64_t)k * nthr;
      const bool right = pp[k] >= 128;
      const int x = (int)(pp[k] & 127u);
      const uint64_t* w = right ? b[k] : a[k];
      uint32_t cnt = qd_count(w, cc[k], x, right ? 0ull : ~0ull);
      uint64_t dw = (cc[k] & 2u) ? a[k][1] : a[k][0];
      uint64_t delta = (dw >> (16 * (cc[k] & 1u))) & 0xffffull;        // u16 slot c + (c & 2)
      uint64_t base = ((uint64_t)s[k] << QD_SHIFT) + delta;
      uint64_t r = right ? base + cnt : base - cnt;
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
}

// rank_4: three plane popcounts per word pair give all four symbols
// (L = #low-bit-set, H = #high-bit-set, T = #both; A = len - L - H + T, C = L - T, G = H - T).
template <int K, bool SMALLQ>
__global__ void __launch_bounds__(256) k_qd_all4(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                 const uint64_t* __restrict__ q, uint64_t* __restrict__ out4,
                                                 uint64_t m, uint64_t last_line) {
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t qn[K];
  uint32_t cn[K];
  qd_load_group<K, false>(q, nullptr, i0, nthr, m, qn, cn);
  for (; i0 < m; i0 += nthr * K) {
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    qd_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t a[K][4], b[K][4];
    uint4 s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint4* ln = lines + 4 * jj[k];
      ld_sector_na(ln, a[k][0], a[k][1], a[k][2], a[k][3]);
      b[k][0] = b[k][1] = b[k][2] = b[k][3] = 0;
      if (pp[k] >= 128) ld_sector_na(ln + 2, b[k][0], b[k][1], b[k][2], b[k][3]);
      s[k] = __ldg(reinterpret_cast<const uint4*>(super) + (jj[k] >> QD_SB_LOG));
    }
    qd_load_group<K, false>(q, nullptr, i0 + nthr * K, nthr, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint64_t idx = i0 + (uint64_t)k * nthr;
      const bool right = pp[k] >= 128;
      const int x = (int)(pp[k] & 127u);
      const uint64_t inv = right ? 0ull : ~0ull;
      const uint64_t* w = right ? b[k] : a[k];
      uint32_t nl = 0, nh = 0, nt = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        uint64_t msk = prefix_mask(x, t) ^ inv;
        uint64_t l = ~w[2 * t] & msk, hh = ~w[2 * t + 1] & msk;   // planes store the negation
        nl += __popcll(l);
        nh += __popcll(hh);
        nt += __popcll(l & hh);
      }
      const uint32_t len = right ? (uint32_t)x : 128u - (uint32_t)x;   // |p - 128| masked chars
      uint32_t cnt[4] = {len - nl - nh + nt, nl - nt, nh - nt, nt};
      uint32_t sv[4] = {s[k].x, s[k].y, s[k].z, s[k].w};
      uint64_t r[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint64_t dw = (c & 2) ? a[k][1] : a[k][0];
        uint64_t delta = (dw >> (16 * (c & 1))) & 0xffffull;
        uint64_t base = ((uint64_t)sv[c] << QD_SHIFT) + delta;
        r[c] = right ? base + cnt[c] : base - cnt[c];
      }
      if (idx < m) st_stream_v4u64(out4 + 4 * idx, r[0], r[1], r[2], r[3]);
    }
  }
}

template <int K, bool SMALLQ, int MODE>
__global__ void __launch_bounds__(256) k_qd_gather(const uint4* __restrict__ lines, const uint64_t* __restrict__ q,
                                                   uint64_t* __restrict__ out, uint64_t m, uint64_t last_line) {
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t qn[K];
  uint32_t cn[K];
  qd_load_group<K, false>(q, nullptr, i0, nthr, m, qn, cn);
  for (; i0 < m; i0 += nthr * K) {
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    qd_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t a[K][4], b[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint4* ln = lines + 4 * jj[k];
      ld_sector_na(ln, a[k][0], a[k][1], a[k][2], a[k][3]);
      b[k][0] = b[k][1] = b[k][2] = b[k][3] = 0;
      if (MODE == 1 || pp[k] >= 128) ld_sector_na(ln + 2, b[k][0], b[k][1], b[k][2], b[k][3]);
    }
    qd_load_group<K, false>(q, nullptr, i0 + nthr * K, nthr, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint64_t idx = i0 + (uint64_t)k * nthr;
      uint64_t r = a[k][0] ^ a[k][1] ^ a[k][2] ^ a[k][3] ^ b[k][0] ^ b[k][1] ^ b[k][2] ^ b[k][3];
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
}

// ---- lane-pair variants: one L2 request per query (see k_bi_rank2 in birank.cu) ------------
// lane 2i loads sector 0 (deltas + data chars [0,96)), lane 2i+1 loads sector 1 (data chars
// [96,224)) only for queries right of the anchor; both loads are in the same warp instruction,
// so the L1 sends one request per 64-B line.  Each lane counts its own case of Listing 1.
template <int K, bool SMALLQ, bool DYN, uint32_t S_LANE = 1>
__global__ void __launch_bounds__(256) k_qd_rank2(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                  const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                                  uint64_t* __restrict__ out, uint64_t m, uint64_t last_line,
                                                  unsigned long long* ctr) {
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = sc_unit_in_warp<16>();
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t i0 = sc.gb + pw, npair = sc.stride;
  uint64_t qn[K];
  uint32_t cn[K];
  qd_load_group<K, true>(q, cs, i0, npair, m, qn, cn);
  while (sc.gb < m) {
    i0 = sc.gb + pw;
    npair = sc.stride;
    uint64_t qq[K], jj[K];
    uint32_t pp[K], cc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { qq[k] = qn[k]; cc[k] = cn[k]; }
    qd_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t w[K][4];
    uint32_t s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (half == 0 || pp[k] >= 128) ld_sector_na(lines + 4 * jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      s[k] = half == S_LANE ? __ldg(super + 4 * (jj[k] >> QD_SB_LOG) + cc[k]) : 0u;
    }
    sc = sc_next<K, DYN, 16>(sc, ctr);
    qd_load_group<K, true>(q, cs, sc.gb + pw, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * npair;
      const bool right = pp[k] >= 128;
      const bool mine = half ? right : !right;
      uint32_t cnt = qd_count(w[k], cc[k], (int)(pp[k] & 127u), half ? 0ull : ~0ull);
      cnt = mine ? cnt : 0u;
      uint64_t dw = (cc[k] & 2u) ? w[k][1] : w[k][0];
      uint64_t delta = (dw >> (16 * (cc[k] & 1u))) & 0xffffull;        // u16 slot c + (c & 2)
      // lane 0: delta - (left count); lane 1: + (right count); 2^13 s from the lane that loaded it
      uint64_t v = (half ? (uint64_t)cnt : delta - cnt) + ((uint64_t)s[k] << QD_SHIFT);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (half == 0 && idx < m) st_stream_u64(out + idx, v);
    }
  }
}

template <int K, bool SMALLQ, bool DYN>
__global__ void __launch_bounds__(256) k_qd_all4_2(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                   const uint64_t* __restrict__ q, uint64_t* __restrict__ out4,
                                                   uint64_t m, uint64_t last_line, unsigned long long* ctr) {
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = sc_unit_in_warp<16>();
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t i0 = sc.gb + pw, npair = sc.stride;
  uint64_t qn[K];
  uint32_t cn[K];
  qd_load_group<K, false>(q, nullptr, i0, npair, m, qn, cn);
  while (sc.gb < m) {
    i0 = sc.gb + pw;
    npair = sc.stride;
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    qd_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t w[K][4];
    uint2 s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (half == 0 || pp[k] >= 128) ld_sector_na(lines + 4 * jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      // lane 0 reads s_A, s_C and lane 1 s_G, s_T: one 16-B segment, one request for the pair
      s[k] = __ldg(reinterpret_cast<const uint2*>(super) + 2 * (jj[k] >> QD_SB_LOG) + half);
    }
    sc = sc_next<K, DYN, 16>(sc, ctr);
    qd_load_group<K, false>(q, nullptr, sc.gb + pw, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * npair;
      const bool right = pp[k] >= 128;
      const int x = (int)(pp[k] & 127u);
      const uint64_t inv = half ? 0ull : ~0ull;
      uint32_t nl = 0, nh = 0, nt = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        uint64_t msk = prefix_mask(x, t) ^ inv;
        uint64_t l = ~w[k][2 * t] & msk, hh = ~w[k][2 * t + 1] & msk;   // planes store the negation
        nl += __popcll(l);
        nh += __popcll(hh);
        nt += __popcll(l & hh);
      }
      const uint32_t len = half ? (uint32_t)x : 128u - (uint32_t)x;
      // four counts <= 128 packed in 8-bit fields: A | C << 8 | G << 16 | T << 24
      const uint32_t packed = (len - nl - nh + nt) | ((nl - nt) << 8) | ((nh - nt) << 16) | (nt << 24);
      const uint32_t other = __shfl_xor_sync(0xffffffffu, packed, 1);
      // lane 1 needs b_G | b_T << 16 (low half of sector-0 word 1, held by lane 0)
      const uint32_t dgt = __shfl_xor_sync(0xffffffffu, (uint32_t)w[k][1], 1);
      // each lane finishes two of the four symbols: lane 0 -> A, C; lane 1 -> G, T
      const uint32_t cnt = (right == (half == 1)) ? packed : other;     // the counting lane's packed counts
      const uint32_t dl = half ? dgt : (uint32_t)w[k][0];
      const uint32_t c0 = (cnt >> (16 * half)) & 0xffu, c1 = (cnt >> (16 * half + 8)) & 0xffu;
      const uint64_t b0 = ((uint64_t)s[k].x << QD_SHIFT) + (dl & 0xffffu);
      const uint64_t b1 = ((uint64_t)s[k].y << QD_SHIFT) + (dl >> 16);
      const uint64_t r0 = right ? b0 + c0 : b0 - c0, r1 = right ? b1 + c1 : b1 - c1;
      if (idx < m) asm volatile("st.global.L1::no_allocate.v2.u64 [%0], {%1,%2};" ::"l"(out4 + 4 * idx + 2 * half),
                                "l"(r0), "l"(r1) : "memory");
    }
  }
}

template <int K, bool SMALLQ, int MODE, bool DYN>
__global__ void __launch_bounds__(256) k_qd_gather2(const uint4* __restrict__ lines, const uint64_t* __restrict__ q,
                                                    uint64_t* __restrict__ out, uint64_t m, uint64_t last_line,
                                                    unsigned long long* ctr) {
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = sc_unit_in_warp<16>();
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t i0 = sc.gb + pw, npair = sc.stride;
  uint64_t qn[K];
  uint32_t cn[K];
  qd_load_group<K, false>(q, nullptr, i0, npair, m, qn, cn);
  while (sc.gb < m) {
    i0 = sc.gb + pw;
    npair = sc.stride;
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    qd_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t w[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (MODE == 1 || half == 0 || pp[k] >= 128)
        ld_sector_na(lines + 4 * jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
    }
    sc = sc_next<K, DYN, 16>(sc, ctr);
    qd_load_group<K, false>(q, nullptr, sc.gb + pw, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * npair;
      if (MODE == 4) {          // rank_4's output shape: each lane of the pair stores 16 B (32 B per query)
        const uint64_t a = w[k][0] ^ w[k][1], b = w[k][2] ^ w[k][3];
        if (idx < m) asm volatile("st.global.L1::no_allocate.v2.u64 [%0], {%1,%2};" ::"l"(out + 4 * idx + 2 * half),
                                  "l"(a), "l"(b) : "memory");
        continue;
      }
      uint64_t v = w[k][0] ^ w[k][1] ^ w[k][2] ^ w[k][3];
      v ^= __shfl_xor_sync(0xffffffffu, v, 1);
      if (half == 0 && idx < m) st_stream_u64(out + idx, v);
    }
  }
}

extern int g_rank_k;
extern int g_rank_blocks_per_sm;
extern int g_rank_pair;
extern int g_rank_lane_table;
extern int g_index64;
extern int g_rank_smem;

template <int K>
static unsigned qd_grid(const qr_index* h, uint64_t m, bool pair) {
  const uint64_t per_thread = pair ? K : 2 * K;
  return grid_stride_blocks((2 * m + per_thread - 1) / per_thread, 256, h->sm_count, g_rank_blocks_per_sm);
}
template <int K>
static cudaError_t qd_rank_k(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                             bool pair, cudaStream_t st) {
  unsigned g = qd_grid<K>(h, m, pair);
  const uint64_t last = h->n_lines - 1;
  const bool small = h->n < (1ull << 37) && !g_index64;
  if (pair) {
    const bool dyn = use_dyn_order(m);
    const uint4* L = h->lines;
    const uint32_t* S = h->super;
    if (small) return launch_ordered(k_qd_rank2<K, true, false>, k_qd_rank2<K, true, true>, dyn, h->device, h->sm_count,
                                     g, st, L, S, q, c, out, m, last);
    return launch_ordered(k_qd_rank2<K, false, false>, k_qd_rank2<K, false, true>, dyn, h->device, h->sm_count, g, st,
                          L, S, q, c, out, m, last);
  } else {
    if (small) k_qd_rank<K, true><<<g, 256, 0, st>>>(h->lines, h->super, q, c, out, m, last);
    else       k_qd_rank<K, false><<<g, 256, 0, st>>>(h->lines, h->super, q, c, out, m, last);
  }
  return cudaGetLastError();
}
template <int K>
static cudaError_t qd_all4_k(const qr_index* h, const uint64_t* q, uint64_t* out4, uint64_t m, bool pair,
                             cudaStream_t st) {
  unsigned g = qd_grid<K>(h, m, pair);
  const uint64_t last = h->n_lines - 1;
  const bool small = h->n < (1ull << 37) && !g_index64;
  if (pair) {
    const bool dyn = use_dyn_order(m);
    const uint4* L = h->lines;
    const uint32_t* S = h->super;
    if (small) return launch_ordered(k_qd_all4_2<K, true, false>, k_qd_all4_2<K, true, true>, dyn, h->device,
                                     h->sm_count, g, st, L, S, q, out4, m, last);
    return launch_ordered(k_qd_all4_2<K, false, false>, k_qd_all4_2<K, false, true>, dyn, h->device, h->sm_count, g, st,
                          L, S, q, out4, m, last);
  } else {
    if (small) k_qd_all4<K, true><<<g, 256, 0, st>>>(h->lines, h->super, q, out4, m, last);
    else       k_qd_all4<K, false><<<g, 256, 0, st>>>(h->lines, h->super, q, out4, m, last);
  }
  return cudaGetLastError();
}
template <int K>
static cudaError_t qd_gather_k(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode,
                               cudaStream_t st) {
  unsigned g = qd_grid<K>(h, m, g_rank_pair != 0);
  const uint64_t last = h->n_lines - 1;
  const bool small = h->n < (1ull << 37) && !g_index64;
  if (mode == 2) mode = 0;   // (superblock-inclusive ceiling: BiRank only)
  if (g_rank_pair) {
    const bool dyn = use_dyn_order(m);
    const uint4* L = h->lines;
    const int dev = h->device, sms = h->sm_count;
#define QR_QG2(SQ, MO) launch_ordered(k_qd_gather2<K, SQ, MO, false>, k_qd_gather2<K, SQ, MO, true>, dyn, dev, sms, g, st, \
                                      L, q, out, m, last)
    if (mode == 4) return small ? QR_QG2(true, 4) : QR_QG2(false, 4);
    if (small) return mode ? QR_QG2(true, 1) : QR_QG2(true, 0);
    return mode ? QR_QG2(false, 1) : QR_QG2(false, 0);
#undef QR_QG2
  }
  if (mode == 4) return cudaErrorNotSupported;   // the rank_4-shaped ceiling exists for lane pairs only
  if (small) {
    if (mode) k_qd_gather<K, true, 1><<<g, 256, 0, st>>>(h->lines, q, out, m, last);
    else      k_qd_gather<K, true, 0><<<g, 256, 0, st>>>(h->lines, q, out, m, last);
  } else {
    if (mode) k_qd_gather<K, false, 1><<<g, 256, 0, st>>>(h->lines, q, out, m, last);
    else      k_qd_gather<K, false, 0><<<g, 256, 0, st>>>(h->lines, q, out, m, last);
  }
  return cudaGetLastError();
}

cudaError_t launch_quadrank_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                 cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  if (h->spack_big && g_rank_smem != 0 && m >= (1ull << 22) && !g_index64) return launch_big_pack_qd(h, q, c, out, m, 0, st);
  const int shape = rank_shape(h, m);
  if (shape == RANK_CLUSTER) return launch_super_pack_rank(h, q, c, out, m, 0, st);
  if (shape == RANK_LANE && g_rank_lane_table) {
    const cudaError_t e = launch_lane_table_rank(h, q, c, out, m, 0, st);
    if (e != cudaErrorNotSupported) return e;
  }
  const bool pair = shape == RANK_PAIR;
  switch (g_rank_k) {
    case 1: return qd_rank_k<1>(h, q, c, out, m, pair, st);
    case 2: return qd_rank_k<2>(h, q, c, out, m, pair, st);
    case 8: return qd_rank_k<8>(h, q, c, out, m, pair, st);
    default: return qd_rank_k<4>(h, q, c, out, m, pair, st);
  }
}
cudaError_t launch_quadrank_all4(const qr_index* h, const uint64_t* q, uint64_t* out4, uint64_t m, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  if (h->spack_big && g_rank_smem != 0 && m >= (1ull << 22) && !g_index64) return launch_big_pack_qd(h, q, nullptr, out4, m, 1, st);
  const int shape = rank_shape(h, m);
  if (shape == RANK_CLUSTER) return launch_super_pack_rank(h, q, nullptr, out4, m, 1, st);
  if (shape == RANK_LANE && g_rank_lane_table) {
    const cudaError_t e = launch_lane_table_rank(h, q, nullptr, out4, m, 1, st);
    if (e != cudaErrorNotSupported) return e;
  }
  const bool pair = shape == RANK_PAIR;
  switch (g_rank_k) {
    case 1: return qd_all4_k<1>(h, q, out4, m, pair, st);
    case 2: return qd_all4_k<2>(h, q, out4, m, pair, st);
    case 8: return qd_all4_k<8>(h, q, out4, m, pair, st);
    default: return qd_all4_k<4>(h, q, out4, m, pair, st);
  }
}
cudaError_t launch_qd_gather(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode,
                             cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  switch (g_rank_k) {
    case 1: return qd_gather_k<1>(h, q, out, m, mode, st);
    case 2: return qd_gather_k<2>(h, q, out, m, mode, st);
    case 8: return qd_gather_k<8>(h, q, out, m, mode, st);
    default: return qd_gather_k<4>(h, q, out, m, mode, st);
  }
}

}  // namespace qr
