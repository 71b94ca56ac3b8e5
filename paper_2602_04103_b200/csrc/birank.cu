// birank.cu — BiRank16 (sigma = 2) on sm_100a: layout builder and the rank(q) kernel.
//
// Layout (§3; R2, R4): line j is 64 B = 32 u16:
//   u16[0] = b_j = rank(jB + 240) - 2^11 s_{j>>7}
//   u16[1..31] = text u16 words [31j, 31j+31)            (496 = 31*16 data bits)
// so line bit 16+k is data bit k, and the anchor (data bit 240) is line bit 256: the
// first 32-B sector holds b_j and data bits [0,240), the second holds data bits [240,496).
// Superblocks: s_i = floor(rank(128 i B) / 2^11) as u32.
//
// Query (Eq. 1): j = q / 496, p = 16 + q - 496 j in [16, 512);
//   p <  256: rank = 2^11 s + b_j - popc(line bits [p, 256))     (sector 0 only)
//   p >= 256: rank = 2^11 s + b_j + popc(line bits [256, p))     (sectors 0 and 1)
#include <cub/device/device_scan.cuh>

#include "qr_common.cuh"
#include "sched.cuh"

namespace qr {

// ------------------------------------------------------------------ build

// Per line: c1 = popc(data bits [0,240)) = 15 text u16 words, tot = popc(all 496 data bits).
__global__ void k_bi_count(const uint16_t* __restrict__ t16, uint64_t L, uint32_t* __restrict__ c1,
                           uint64_t* __restrict__ tot) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint16_t* p = t16 + 31 * j;
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int k = 0; k < 15; ++k) lo += __popc((uint32_t)p[k]);
#pragma unroll
    for (int k = 15; k < 31; ++k) hi += __popc((uint32_t)p[k]);
    c1[j] = lo;
    tot[j] = lo + hi;
  }
}

// R = exclusive prefix of tot (R_j = rank(jB)); writes s_i and the lines.
__global__ void k_bi_write(const uint16_t* __restrict__ t16, uint64_t L, const uint32_t* __restrict__ c1,
                           const uint64_t* __restrict__ R, uint4* __restrict__ lines, uint32_t* __restrict__ super) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t sb = R[(j >> BI_SB_LOG) << BI_SB_LOG] >> BI_SHIFT;        // s_{j>>7}
    if ((j & ((1u << BI_SB_LOG) - 1)) == 0) super[j >> BI_SB_LOG] = (uint32_t)sb;
    uint32_t b = (uint32_t)(R[j] + c1[j] - (sb << BI_SHIFT));         // rank(jB+240) - 2^11 s
    const uint16_t* p = t16 + 31 * j;
    uint32_t u[16];
    u[0] = b | ((uint32_t)p[0] << 16);
#pragma unroll
    for (int k = 1; k < 16; ++k) u[k] = (uint32_t)p[2 * k - 1] | ((uint32_t)p[2 * k] << 16);
    uint4* dst = lines + 4 * j;
#pragma unroll
    for (int v = 0; v < 4; ++v) dst[v] = make_uint4(u[4 * v], u[4 * v + 1], u[4 * v + 2], u[4 * v + 3]);
  }
}

__global__ void k_mask_tail_bits(uint64_t* words, uint64_t n) {
  uint64_t r = n & 63;
  if (r) words[n >> 6] &= (1ull << r) - 1ull;
}

qr_status birank_build_device(const uint64_t* d_bits, uint64_t n, int device, cudaStream_t st, qr_index** out) {
  // d_bits: device copy owned by the caller (api.cu), >= max(62 L, 8 ceil(n/64)) bytes, zero padded.
  qr_index* h = nullptr;
  qr_status rs = alloc_index(2, n, device, &h);
  if (rs != QR_OK) return rs;
  const uint64_t L = h->n_lines;
  uint32_t* c1 = nullptr;
  uint64_t *tot = nullptr, *R = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cudaSuccess;
  auto bail = [&](cudaError_t err, const char* what) {
    cudaFreeAsync(c1, st); cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(tmp, st);
    qr_free(h);
    return cuda_fail(err, what);
  };
  k_mask_tail_bits<<<1, 1, 0, st>>>(const_cast<uint64_t*>(d_bits), n);
  if ((e = cudaMallocAsync((void**)&c1, L * sizeof(uint32_t), st))) return bail(e, "alloc c1");
  if ((e = cudaMallocAsync((void**)&tot, L * sizeof(uint64_t), st))) return bail(e, "alloc tot");
  if ((e = cudaMallocAsync((void**)&R, L * sizeof(uint64_t), st))) return bail(e, "alloc R");
  const int sms = h->sm_count;
  unsigned g = grid_stride_blocks(L, 256, sms, 16);
  k_bi_count<<<g, 256, 0, st>>>(reinterpret_cast<const uint16_t*>(d_bits), L, c1, tot);
  if ((e = cudaGetLastError())) return bail(e, "k_bi_count");
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, tot, R, (int64_t)L, st))) return bail(e, "scan size");
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st))) return bail(e, "alloc scan tmp");
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, tot, R, (int64_t)L, st))) return bail(e, "scan");
  k_bi_write<<<g, 256, 0, st>>>(reinterpret_cast<const uint16_t*>(d_bits), L, c1, R, h->lines, h->super);
  if ((e = cudaGetLastError())) return bail(e, "k_bi_write");
  cudaFreeAsync(c1, st); cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(tmp, st);
  if ((rs = build_super_pack(h, st)) != QR_OK) { qr_free(h); return rs; }
  *out = h;
  return QR_OK;
}

// ------------------------------------------------------------------ rank

template <bool SMALLQ>
__device__ __forceinline__ uint64_t bi_line_of(uint64_t q) {
  if (SMALLQ) return (uint64_t)((uint32_t)(q >> 4) / 31u);   // floor(floor(q/16)/31) = floor(q/496), q < 2^36
  return q / BI_B;
}

// K independent queries per thread per group: all K line gathers are issued before any
// popcount, and the next group's K query positions are loaded while those gathers are in
// flight (software pipelining of the dependent q -> line chain), so a thread keeps K line
// misses outstanding nearly all the time.  Grid = SM count x CTAs/SM, grid-stride over the
// query array (coalesced q loads and out stores).
template <int K, bool SMALLQ>
__device__ __forceinline__ void bi_locate(const uint64_t (&qq)[K], uint64_t last_line, uint64_t (&jj)[K],
                                          uint32_t (&pp)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uint64_t j = bi_line_of<SMALLQ>(qq[k]);
    j = j > last_line ? last_line : j;                   // q > n: memory-safe clamp
    uint64_t p = 16 + qq[k] - j * BI_B;
    pp[k] = p > 511 ? 511u : (uint32_t)p;
    jj[k] = j;
  }
}

template <int K>
__device__ __forceinline__ void load_q_group(const uint64_t* __restrict__ q, uint64_t i0, uint64_t nthr, uint64_t m,
                                             uint64_t (&qn)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uint64_t idx = i0 + (uint64_t)k * nthr;
    qn[k] = idx < m ? ld_stream_u64(q + idx) : 0;
  }
}

template <int K, bool SMALLQ, bool HAS_C>
__global__ void __launch_bounds__(256) k_bi_rank(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                 const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                                 uint64_t* __restrict__ out, uint64_t m, uint64_t last_line) {
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t qn[K];
  load_q_group<K>(q, i0, nthr, m, qn);
  for (; i0 < m; i0 += nthr * K) {
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    bi_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t a[K][4], b[K][4];
    uint32_t s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint4* ln = lines + 4 * jj[k];
      ld_sector_na(ln, a[k][0], a[k][1], a[k][2], a[k][3]);
      b[k][0] = b[k][1] = b[k][2] = b[k][3] = 0;
      if (pp[k] >= 256) ld_sector_na(ln + 2, b[k][0], b[k][1], b[k][2], b[k][3]);
      s[k] = __ldg(super + (jj[k] >> BI_SB_LOG));
    }
    load_q_group<K>(q, i0 + nthr * K, nthr, m, qn);      // next group, overlapping the gathers
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint64_t idx = i0 + (uint64_t)k * nthr;
      const bool right = pp[k] >= 256;
      const int x = (int)(pp[k] & 255u);                  // p (left) or p - 256 (right)
      const uint64_t inv = right ? 0ull : ~0ull;          // left: suffix [p,256) = ~prefix(p)
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint64_t w = right ? b[k][t] : a[k][t];
        cnt += __popcll(w & (prefix_mask(x, t) ^ inv));
      }
      // left queries have p >= 16, so the inverted prefix never covers line bits [0,16) = b_j.
      uint64_t base = ((uint64_t)s[k] << BI_SHIFT) + (a[k][0] & 0xffffull);
      uint64_t r = right ? base + cnt : base - cnt;
      if (HAS_C) {
        if (idx < m && cs[idx] == 0) r = qq[k] - r;
      }
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
}

// Gather ceiling (G9): identical q stream (same pipelining), line arithmetic and sector
// loads; no popcount, no superblock read.  MODE 0: the sectors rank reads; MODE 1: the full line.
template <int K, bool SMALLQ, int MODE>
__global__ void __launch_bounds__(256) k_bi_gather(const uint4* __restrict__ lines, const uint64_t* __restrict__ q,
                                                   uint64_t* __restrict__ out, uint64_t m, uint64_t last_line) {
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t qn[K];
  load_q_group<K>(q, i0, nthr, m, qn);
  for (; i0 < m; i0 += nthr * K) {
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    bi_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t a[K][4], b[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint4* ln = lines + 4 * jj[k];
      ld_sector_na(ln, a[k][0], a[k][1], a[k][2], a[k][3]);
      b[k][0] = b[k][1] = b[k][2] = b[k][3] = 0;
      if (MODE == 1 || pp[k] >= 256) ld_sector_na(ln + 2, b[k][0], b[k][1], b[k][2], b[k][3]);
    }
    load_q_group<K>(q, i0 + nthr * K, nthr, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint64_t idx = i0 + (uint64_t)k * nthr;
      uint64_t r = a[k][0] ^ a[k][1] ^ a[k][2] ^ a[k][3] ^ b[k][0] ^ b[k][1] ^ b[k][2] ^ b[k][3];
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
}

// ---- lane-pair variants: one L2 request per query ---------------------------------------
// Every random sector load is one L2 request, and on B200 the random-miss path saturates at
// ~45 G requests/s whatever the request size (tools/gather_probe: 4 B to 32 B loads all run
// at the same rate).  So the two sectors of a query are loaded by two lanes of the SAME warp
// instruction (lane 2i: sector 0 with b_j and data bits [0,240); lane 2i+1: sector 1, only
// when q lies right of the anchor): the L1 merges them into ONE request for the 64-B line
// with a two-sector mask, i.e. 1 request per query instead of 1.52.  Each lane counts its own
// half (Eq. 1's two cases are exactly the two sectors) and one shuffle adds the halves.
// Loop bounds are warp-uniform so that the shuffle sees every lane.
template <int K, bool SMALLQ, bool HAS_C, uint32_t S_LANE, bool DYN>
__global__ void __launch_bounds__(256) k_bi_rank2(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                  const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                                  uint64_t* __restrict__ out, uint64_t m, uint64_t last_line,
                                                  unsigned long long* ctr) {
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = sc_unit_in_warp<16>();
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t i0 = sc.gb + pw, npair = sc.stride;                      // first pair of this warp (uniform)
  uint64_t qn[K];
  load_q_group<K>(q, i0, npair, m, qn);
  while (sc.gb < m) {
    i0 = sc.gb + pw;
    npair = sc.stride;
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    bi_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t w[K][4];
    uint32_t s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (half == 0 || pp[k] >= 256) ld_sector_na(lines + 4 * jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      s[k] = half == S_LANE ? __ldg(super + (jj[k] >> BI_SB_LOG)) : 0u;
    }
    sc = sc_next<K, DYN, 16>(sc, ctr);
    load_q_group<K>(q, sc.gb + pw, sc.stride, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * npair;
      const bool right = pp[k] >= 256;
      const int x = (int)(pp[k] & 255u);
      const bool mine = half ? right : !right;            // which case of Eq. 1 this lane counts
      const uint64_t inv = half ? 0ull : ~0ull;           // lane 0: suffix [p,256); lane 1: prefix [256,p)
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) cnt += __popcll(w[k][t] & (prefix_mask(x, t) ^ inv));
      cnt = mine ? cnt : 0u;
      // lane 0: b_j - (left count); lane 1: + (right count); 2^11 s from the lane that loaded it
      uint64_t v = (half ? (uint64_t)cnt : (w[k][0] & 0xffffull) - cnt) + ((uint64_t)s[k] << BI_SHIFT);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (HAS_C) {
        if (half == 0 && idx < m && cs[idx] == 0) v = qq[k] - v;
      }
      if (half == 0 && idx < m) st_stream_u64(out + idx, v);
    }
  }
}

// (S_LANE: the pair lane that loads the superblock word; lane 1 — idle for the 48% of queries
// left of the anchor — measured 36.9 vs 35.6 Gq/s for lane 0 on configs[1], profiles/r01_s_probe.)
// Gather ceiling with the same lane-pair loads (MODE 0: the sectors rank2 reads; MODE 1: both
// sectors always; MODE 2: the sectors rank2 reads plus its superblock-word load).
template <int K, bool SMALLQ, int MODE, bool DYN>
__global__ void __launch_bounds__(256) k_bi_gather2(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                    const uint64_t* __restrict__ q, uint64_t* __restrict__ out, uint64_t m,
                                                    uint64_t last_line, unsigned long long* ctr) {
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = sc_unit_in_warp<16>();
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t i0 = sc.gb + pw, npair = sc.stride;
  uint64_t qn[K];
  load_q_group<K>(q, i0, npair, m, qn);
  while (sc.gb < m) {
    i0 = sc.gb + pw;
    npair = sc.stride;
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    bi_locate<K, SMALLQ>(qq, last_line, jj, pp);
    uint64_t w[K][4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (MODE == 1 || half == 0 || pp[k] >= 256)
        ld_sector_na(lines + 4 * jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      if (MODE == 2 && half == 0) w[k][0] ^= __ldg(super + (jj[k] >> BI_SB_LOG));
    }
    sc = sc_next<K, DYN, 16>(sc, ctr);
    load_q_group<K>(q, sc.gb + pw, sc.stride, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * npair;
      uint64_t v = w[k][0] ^ w[k][1] ^ w[k][2] ^ w[k][3];
      v ^= __shfl_xor_sync(0xffffffffu, v, 1);
      if (half == 0 && idx < m) st_stream_u64(out + idx, v);
    }
  }
}

extern int g_rank_k;              // tuning knobs (api.cu)
extern int g_rank_blocks_per_sm;
extern int g_rank_pair;
extern int g_rank_lane_table;
extern int g_index64;
extern int g_rank_smem;
extern int g_rank_s_lane;

template <int K>
static cudaError_t bi_rank_k(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                             bool pair, cudaStream_t st) {
  const bool small = h->n < (1ull << 36) && !g_index64;
  const uint64_t per_thread = pair ? K : 2 * K;          // pair kernels: 2 threads per query
  unsigned g = grid_stride_blocks((2 * m + per_thread - 1) / per_thread, 256, h->sm_count, g_rank_blocks_per_sm);
  const uint64_t last = h->n_lines - 1;
  if (pair) {
    const bool s0 = g_rank_s_lane == 0;
    const bool dyn = use_dyn_order(m);
    const int dev = h->device, sms = h->sm_count;
#define QR_BI2(SQ, HC, SL) launch_ordered(k_bi_rank2<K, SQ, HC, SL, false>, k_bi_rank2<K, SQ, HC, SL, true>, dyn, dev, sms, \
                                          g, st, (const uint4*)h->lines, (const uint32_t*)h->super, q, c, out, m, last)
    if (small) {
      if (c) return QR_BI2(true, true, 1);
      if (s0) return QR_BI2(true, false, 0);
      return QR_BI2(true, false, 1);
    }
    if (c) return QR_BI2(false, true, 1);
    return QR_BI2(false, false, 1);
#undef QR_BI2
  }
  if (small) {
    if (c) k_bi_rank<K, true, true><<<g, 256, 0, st>>>(h->lines, h->super, q, c, out, m, last);
    else   k_bi_rank<K, true, false><<<g, 256, 0, st>>>(h->lines, h->super, q, c, out, m, last);
  } else {
    if (c) k_bi_rank<K, false, true><<<g, 256, 0, st>>>(h->lines, h->super, q, c, out, m, last);
    else   k_bi_rank<K, false, false><<<g, 256, 0, st>>>(h->lines, h->super, q, c, out, m, last);
  }
  return cudaGetLastError();
}

cudaError_t launch_birank_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                               cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  // n >= 2^35 (or forced for tests): superblock words from a CS-CTA cluster table (sbcache.cu)
  if (h->spack_big && g_rank_smem != 0 && m >= (1ull << 22) && !g_index64) return launch_big_pack_rank(h, q, c, out, m, st);
  const int shape = rank_shape(h, m);
  if (shape == RANK_CLUSTER) return launch_super_pack_rank(h, q, c, out, m, 0, st);
  if (shape == RANK_LANE && g_rank_lane_table) {
    const cudaError_t e = launch_lane_table_rank(h, q, c, out, m, 0, st);
    if (e != cudaErrorNotSupported) return e;
  }
  const bool pair = shape == RANK_PAIR;
  switch (g_rank_k) {
    case 1: return bi_rank_k<1>(h, q, c, out, m, pair, st);
    case 2: return bi_rank_k<2>(h, q, c, out, m, pair, st);
    case 8: return bi_rank_k<8>(h, q, c, out, m, pair, st);
    default: return bi_rank_k<4>(h, q, c, out, m, pair, st);
  }
}

template <int K>
static cudaError_t bi_gather_k(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode,
                               cudaStream_t st) {
  const bool small = h->n < (1ull << 36) && !g_index64;
  const uint64_t per_thread = g_rank_pair ? K : 2 * K;
  unsigned g = grid_stride_blocks((2 * m + per_thread - 1) / per_thread, 256, h->sm_count, g_rank_blocks_per_sm);
  const uint64_t last = h->n_lines - 1;
  if (g_rank_pair) {
    const bool dyn = use_dyn_order(m);
    const int dev = h->device, sms = h->sm_count;
#define QR_BG2(SQ, MO) launch_ordered(k_bi_gather2<K, SQ, MO, false>, k_bi_gather2<K, SQ, MO, true>, dyn, dev, sms, g, st, \
                                      (const uint4*)h->lines, (const uint32_t*)h->super, q, out, m, last)
    if (small) return mode == 2 ? QR_BG2(true, 2) : mode == 1 ? QR_BG2(true, 1) : QR_BG2(true, 0);
    return mode == 2 ? QR_BG2(false, 2) : mode == 1 ? QR_BG2(false, 1) : QR_BG2(false, 0);
#undef QR_BG2
  }
  if (mode == 2) mode = 0;
  if (small) {
    if (mode) k_bi_gather<K, true, 1><<<g, 256, 0, st>>>(h->lines, q, out, m, last);
    else      k_bi_gather<K, true, 0><<<g, 256, 0, st>>>(h->lines, q, out, m, last);
  } else {
    if (mode) k_bi_gather<K, false, 1><<<g, 256, 0, st>>>(h->lines, q, out, m, last);
    else      k_bi_gather<K, false, 0><<<g, 256, 0, st>>>(h->lines, q, out, m, last);
  }
  return cudaGetLastError();
}

cudaError_t launch_bi_gather(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode,
                             cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  switch (g_rank_k) {
    case 1: return bi_gather_k<1>(h, q, out, m, mode, st);
    case 2: return bi_gather_k<2>(h, q, out, m, mode, st);
    case 8: return bi_gather_k<8>(h, q, out, m, mode, st);
    default: return bi_gather_k<4>(h, q, out, m, mode, st);
  }
}

}  // namespace qr
