// bucket.cu — BiRank16 rank(q) for large batches over a structure far larger than the L2:
// queries regrouped by line region so that every line gather is an L2 hit.
//
// The direct kernel (sbcache.cu k_bi_rank2c) answers each query with one random 64-B line
// gather from HBM; at 10^9 queries over the 2.2 GB configs[1] structure it sits at the DRAM
// random-request ceiling (~46 G requests/s), half the streaming bandwidth.  But
// the batch is a set: 10^9 queries over 3.5·10^7 lines read every line ~29 times.  This path
// reorders the work, not the method — each query is still Eq. 1 on its own
// line — in four stream-ordered passes, three of them streaming:
//   1. k_bk_hist     histogram of the queries over NB line regions ("buckets", <= 512, each
//                    2^sh lines, 8-16 MB: a few fit the 126 MB L2 at once);
//   2. k_bk_scatter  the queries regrouped by bucket: entry = (q - bucket base) << 1 | c-bit,
//                    index in the low 32 bits; staged per 8192-query tile in shared memory and
//                    written as runs, so the scatter streams;
//   3. k_bk_rank     buckets in order (dynamic tile counter: the grid works on a few adjacent
//                    buckets at a time, their lines L2-resident), Eq. 1 per entry, and the result
//                    regrouped by destination (2^dsh consecutive output slots per group) the
//                    same way;
//   4. k_bk_unpermute  destination groups in order: out[idx] = result, scattered stores inside a
//                    32 MB window that the L2 merges into full lines before write-back.
// HBM traffic: 8 (hist) + 16 (scatter) + 16 + lines once (rank) + 16 (unpermute) = ~58 GB per
// 10^9 queries instead of ~10^9 random requests.  The caller's `out` doubles as the scatter
// buffer when it does not overlap q or c; one m x 8 B buffer comes from the stream-ordered pool.
#include <mutex>
#include <set>

#include "qr_common.cuh"

namespace qr {

constexpr int BK_T = 8192;                // entries per tile
constexpr int BK_THREADS = 512;
constexpr int BK_PER = BK_T / BK_THREADS; // entries per thread per tile
constexpr int BK_NB_MAX = 512;            // buckets and destination groups (each <= 512)

struct BkGeom {
  uint64_t m;          // queries of this call (< 2^32)
  uint64_t qmax;       // largest q that is kept (q > n: contract violation, clamped)
  uint32_t sh;         // bucket = line >> sh
  uint32_t nb;         // buckets
  uint32_t dsh;        // destination group = index >> dsh
  uint32_t nd;         // destination groups
  uint64_t last_line;
};

// q -> line (q <= qmax < 2^36, so q >> 4 fits 32 bits: floor(q/496) = floor((q>>4)/31))
__device__ __forceinline__ uint32_t bk_line(uint64_t q) { return (uint32_t)(q >> 4) / 31u; }

__global__ void __launch_bounds__(BK_THREADS) k_bk_hist(const uint64_t* __restrict__ q, BkGeom g,
                                                        unsigned int* __restrict__ hist) {
  __shared__ unsigned int h[BK_NB_MAX];
  for (uint32_t i = threadIdx.x; i < g.nb; i += BK_THREADS) h[i] = 0;
  __syncthreads();
  const uint64_t step = (uint64_t)gridDim.x * BK_THREADS * 4;
  for (uint64_t i0 = blockIdx.x * (uint64_t)BK_THREADS * 4 + threadIdx.x; i0 < g.m; i0 += step) {
    uint64_t v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = i0 + (uint64_t)k * BK_THREADS;
      v[k] = i < g.m ? ld_stream_u64(q + i) : ~0ull;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i0 + (uint64_t)k * BK_THREADS < g.m) {
        const uint64_t qq = v[k] < g.qmax ? v[k] : g.qmax;
        atomicAdd(&h[bk_line(qq) >> g.sh], 1u);
      }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < g.nb; i += BK_THREADS)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// starts[b] = exclusive prefix of hist (starts[nb] = m); cur[b] = starts[b]; dcur[d] = d << dsh
__global__ void k_bk_scan(const unsigned int* __restrict__ hist, BkGeom g, unsigned long long* __restrict__ starts,
                          unsigned long long* __restrict__ cur, unsigned long long* __restrict__ dcur) {
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (uint32_t b = 0; b < g.nb; ++b) { starts[b] = s; cur[b] = s; s += hist[b]; }
    starts[g.nb] = s;
  }
  for (uint32_t d = threadIdx.x; d < g.nd; d += blockDim.x) dcur[d] = (unsigned long long)d << g.dsh;
}

// Shared-memory staging of one tile: entries with their group ids are counted per group, the
// tile's runs reserved in the global per-group cursors, placed contiguously and written out run
// by run (consecutive threads, consecutive addresses).
struct BkStage {
  uint64_t* ent;          // [BK_T]
  uint16_t* grp;          // [BK_T]
  unsigned int* cnt;      // [BK_NB_MAX]
  unsigned int* off;      // [BK_NB_MAX]
  unsigned long long* gb; // [BK_NB_MAX]
};

__device__ __forceinline__ void bk_stage_write(const BkStage& S, uint32_t ng, const uint64_t (&e)[BK_PER],
                                               const uint32_t (&gr)[BK_PER], uint32_t valid_mask,
                                               unsigned long long* __restrict__ cur, uint64_t* __restrict__ dst) {
  for (uint32_t i = threadIdx.x; i < ng; i += BK_THREADS) S.cnt[i] = 0;
  __syncthreads();
  uint32_t pos[BK_PER];
#pragma unroll
  for (int k = 0; k < BK_PER; ++k) pos[k] = ((valid_mask >> k) & 1u) ? atomicAdd(&S.cnt[gr[k]], 1u) : 0u;
  __syncthreads();
  // exclusive scan of cnt[0..ng) by warp 0 (ng <= 512: 16 per lane), reservations by all
  if (threadIdx.x < 32) {
    const uint32_t lane = threadIdx.x;
    uint32_t loc[BK_NB_MAX / 32], sum = 0;
#pragma unroll
    for (int t = 0; t < BK_NB_MAX / 32; ++t) {
      const uint32_t i = lane * (BK_NB_MAX / 32) + t;
      loc[t] = i < ng ? S.cnt[i] : 0u;
      sum += loc[t];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += v;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int t = 0; t < BK_NB_MAX / 32; ++t) {
      const uint32_t i = lane * (BK_NB_MAX / 32) + t;
      if (i < ng) S.off[i] = run;
      run += loc[t];
    }
  }
  for (uint32_t i = threadIdx.x; i < ng; i += BK_THREADS)
    if (S.cnt[i]) S.gb[i] = atomicAdd(&cur[i], (unsigned long long)S.cnt[i]);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < BK_PER; ++k)
    if ((valid_mask >> k) & 1u) {
      const uint32_t s = S.off[gr[k]] + pos[k];
      S.ent[s] = e[k];
      S.grp[s] = (uint16_t)gr[k];
    }
  __syncthreads();
  const uint32_t n_in = S.off[ng - 1] + S.cnt[ng - 1];
  for (uint32_t s = threadIdx.x; s < n_in; s += BK_THREADS) {
    const uint32_t b = S.grp[s];
    st_stream_u64(dst + S.gb[b] + (s - S.off[b]), S.ent[s]);
  }
  __syncthreads();
}

__device__ __forceinline__ BkStage bk_stage_carve(unsigned char* smem) {
  BkStage S;
  S.ent = reinterpret_cast<uint64_t*>(smem);
  S.gb = reinterpret_cast<unsigned long long*>(smem + BK_T * 8);
  S.grp = reinterpret_cast<uint16_t*>(smem + BK_T * 8 + BK_NB_MAX * 8);
  S.cnt = reinterpret_cast<unsigned int*>(smem + BK_T * 10 + BK_NB_MAX * 8);
  S.off = S.cnt + BK_NB_MAX;
  return S;
}
constexpr size_t BK_STAGE_SMEM = (size_t)BK_T * 10 + BK_NB_MAX * 16;

template <bool HAS_C>
__global__ void __launch_bounds__(BK_THREADS) k_bk_scatter(const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                                           BkGeom g, unsigned long long* __restrict__ cur,
                                                           uint64_t* __restrict__ A) {
  extern __shared__ __align__(16) unsigned char bk_smem[];
  const BkStage S = bk_stage_carve(bk_smem);
  const uint64_t tiles = (g.m + BK_T - 1) / BK_T;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint64_t base = t * BK_T;
    uint64_t e[BK_PER];
    uint32_t gr[BK_PER], vm = 0;
#pragma unroll
    for (int k = 0; k < BK_PER; ++k) {
      const uint64_t i = base + (uint64_t)k * BK_THREADS + threadIdx.x;
      const bool ok = i < g.m;
      uint64_t qq = ok ? ld_stream_u64(q + i) : 0ull;
      qq = qq < g.qmax ? qq : g.qmax;
      const uint32_t cb = HAS_C ? (ok ? (ld_stream_u8(cs + i) != 0) : 1u) : 1u;
      const uint32_t b = bk_line(qq) >> g.sh;
      const uint64_t ql = qq - (uint64_t)(b << g.sh) * BI_B;            // < 2^sh * 496 < 2^31
      e[k] = (((ql << 1) | cb) << 32) | (uint32_t)i;
      gr[k] = b;
      vm |= (uint32_t)ok << k;
    }
    bk_stage_write(S, g.nb, e, gr, vm, cur, A);
  }
}

template <bool HAS_C>
__global__ void __launch_bounds__(BK_THREADS) k_bk_rank(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                        const uint64_t* __restrict__ A,
                                                        const unsigned long long* __restrict__ starts, BkGeom g,
                                                        unsigned long long* __restrict__ dcur, uint64_t* __restrict__ B,
                                                        unsigned long long* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char bk_smem[];
  const BkStage S = bk_stage_carve(bk_smem);
  __shared__ unsigned long long st_s[BK_NB_MAX + 1];
  __shared__ uint64_t tile_s;
  for (uint32_t i = threadIdx.x; i <= g.nb; i += BK_THREADS) st_s[i] = starts[i];
  const uint64_t tiles = (g.m + BK_T - 1) / BK_T;
  const uint64_t dmask = (1ull << g.dsh) - 1ull;
  while (true) {
    if (threadIdx.x == 0) tile_s = atomicAdd(ctr, 1ull);
    __syncthreads();
    const uint64_t t = tile_s;
    if (t >= tiles) break;
    const uint64_t base = t * BK_T;
    // bucket of the tile's first entry (binary search), then per entry a short forward walk
    uint32_t b0 = 0;
    {
      uint32_t lo = 0, hi = g.nb;                 // largest b with starts[b] <= base
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (st_s[mid] <= base) lo = mid; else hi = mid;
      }
      b0 = lo;
    }
    uint64_t e[BK_PER];
    uint32_t gr[BK_PER], vm = 0;
#pragma unroll
    for (int k0 = 0; k0 < BK_PER; k0 += 4) {
      uint64_t w[4][4], qv[4];
      uint32_t pv[4], sv[4], iv[4], cb[4], bj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t s = base + (uint64_t)(k0 + u) * BK_THREADS + threadIdx.x;
        const bool ok = s < g.m;
        const uint64_t a = ok ? ld_stream_u64(A + s) : 0ull;
        uint32_t b = b0;
        while (b + 1 < g.nb && st_s[b + 1] <= s) ++b;
        cb[u] = (uint32_t)(a >> 32) & 1u;
        iv[u] = (uint32_t)a;
        const uint64_t qq = (uint64_t)(b << g.sh) * BI_B + (a >> 33);
        const uint32_t j = bk_line(qq);
        const uint32_t p = 16u + (uint32_t)(qq - (uint64_t)j * BI_B);   // q <= qmax: j <= last_line, p < 512
        qv[u] = qq;
        pv[u] = p;
        const uint4* L = lines + 4 * (uint64_t)j;
        ld_sector(L, w[u][0], w[u][1], w[u][2], w[u][3]);           // b_j and line bits [0, 256)
        bj[u] = (uint32_t)(w[u][0] & 0xffffull);
        if (p >= 256) ld_sector(L + 2, w[u][0], w[u][1], w[u][2], w[u][3]);   // line bits [256, 512)
        sv[u] = __ldg(super + (j >> BI_SB_LOG));
        vm |= (uint32_t)ok << (k0 + u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t p = pv[u];
        const bool right = p >= 256;
        const int x = (int)(p & 255u);
        const uint64_t inv = right ? 0ull : ~0ull;                  // left: bits [p, 256)
        uint32_t cnt = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) cnt += __popcll(w[u][t] & (prefix_mask(x, t) ^ inv));
        const uint64_t base_r = ((uint64_t)sv[u] << BI_SHIFT) + bj[u];
        uint64_t r = right ? base_r + cnt : base_r - cnt;
        if (HAS_C && !cb[u]) r = qv[u] - r;
        e[k0 + u] = (r << g.dsh) | ((uint64_t)iv[u] & dmask);
        gr[k0 + u] = iv[u] >> g.dsh;
      }
    }
    bk_stage_write(S, g.nd, e, gr, vm, dcur, B);
  }
}

__global__ void __launch_bounds__(BK_THREADS) k_bk_unpermute(const uint64_t* __restrict__ B, BkGeom g,
                                                             uint64_t* __restrict__ out,
                                                             unsigned long long* __restrict__ ctr) {
  __shared__ uint64_t tile_s;
  const uint64_t tiles = (g.m + BK_T - 1) / BK_T;
  const uint64_t dmask = (1ull << g.dsh) - 1ull;
  while (true) {
    if (threadIdx.x == 0) tile_s = atomicAdd(ctr, 1ull);
    __syncthreads();
    const uint64_t t = tile_s;
    __syncthreads();
    if (t >= tiles) break;
    const uint64_t base = t * BK_T;
    uint64_t v[BK_PER];
#pragma unroll
    for (int k = 0; k < BK_PER; ++k) {
      const uint64_t s = base + (uint64_t)k * BK_THREADS + threadIdx.x;
      v[k] = s < g.m ? ld_stream_u64(B + s) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < BK_PER; ++k) {
      const uint64_t s = base + (uint64_t)k * BK_THREADS + threadIdx.x;
      if (s < g.m) out[(s & ~dmask) + (v[k] & dmask)] = v[k] >> g.dsh;   // group d occupies B[d << dsh, ...)
    }
  }
}

int g_rank_bucket = 1;        // 0 never, 1 large batches over structures >> L2, 2 whenever allowed (tests)
int g_rank_bucket_shift = 0;  // 0 auto, else force the bucket shift (tests: many buckets on small n)
int g_rank_bucket_dshift = 0; // 0 auto, else force the destination-group shift (tests)
uint64_t g_rank_bucket_chunk = 1ull << 31;   // queries per bucketed call (indices fit 32 bits)
int l2_bytes(int device);

bool bucket_eligible(const qr_index* h, uint64_t m) {
  if (g_rank_bucket == 0 || h->sigma != 2 || h->layout != QR_LAYOUT_BIRANK16 || h->n >= (1ull << 36)) return false;
  if (g_rank_bucket == 2) return m > 0;
  return m >= (1ull << 24) && (double)h->n_lines * 64.0 >= 4.0 * (double)l2_bytes(h->device);
}

static void bk_pool_keep(int device) {
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> g(mu);
  if (done.count(device)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    // keep up to 24 GB reserved between calls (re-mapping 8 GB per call costs milliseconds)
    uint64_t thr = 24ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done.insert(device);
}

static bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
  return a && b && x < y + nb && y < x + na;
}

static cudaError_t bk_chunk(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                            cudaStream_t st) {
  BkGeom g;
  g.m = m;
  g.last_line = h->n_lines - 1;
  g.qmax = (g.last_line + 1) * BI_B - 1;
  uint32_t sh = 0;
  while (((g.last_line >> sh) + 1) > (uint64_t)BK_NB_MAX) ++sh;
  if (g_rank_bucket_shift > 0 && (uint32_t)g_rank_bucket_shift > sh) sh = (uint32_t)g_rank_bucket_shift;
  g.sh = sh;
  g.nb = (uint32_t)(g.last_line >> sh) + 1;
  uint32_t dsh = 10;
  while (((m - 1) >> dsh) + 1 > (uint64_t)BK_NB_MAX) ++dsh;
  if (g_rank_bucket_dshift > 0 && (uint32_t)g_rank_bucket_dshift > dsh) dsh = (uint32_t)g_rank_bucket_dshift;
  g.dsh = dsh;
  g.nd = (uint32_t)((m - 1) >> dsh) + 1;
  // results must fit 64 - dsh bits (r <= qmax < 2^36) and q - base in 31 bits
  if (dsh > 28 || (((uint64_t)1 << sh) * BI_B) > (1ull << 31)) return cudaErrorNotSupported;

  const int dev = h->device, sms = h->sm_count;
  bk_pool_keep(dev);
  const size_t hdr = 4096 + (size_t)BK_NB_MAX * 32;
  unsigned char* scratch = nullptr;
  uint64_t* A = out;
  const bool alias = overlaps(out, m * 8, q, m * 8) || (c && overlaps(out, m * 8, c, m));
  size_t bytes = hdr + m * 8 + (alias ? m * 8 : 0);
  cudaError_t e = cudaMallocAsync((void**)&scratch, bytes, st);
  if (e) return e;
  unsigned int* hist = reinterpret_cast<unsigned int*>(scratch);                       // [512]
  unsigned long long* starts = reinterpret_cast<unsigned long long*>(scratch + 2048);  // [513]
  unsigned long long* cur = starts + BK_NB_MAX + 8;                                    // [512]
  unsigned long long* dcur = cur + BK_NB_MAX;                                          // [512]
  unsigned long long* ctr = dcur + BK_NB_MAX;                                          // [2]
  uint64_t* B = reinterpret_cast<uint64_t*>(scratch + hdr);
  if (alias) A = B + m;
  e = cudaMemsetAsync(hist, 0, 2048, st);
  if (!e) e = cudaMemsetAsync(ctr, 0, 16, st);
  if (e) { cudaFreeAsync(scratch, st); return e; }
  static_assert(2048 + (BK_NB_MAX + 8) * 8 + 3 * BK_NB_MAX * 8 + 16 <= 4096 + BK_NB_MAX * 32, "header");

  const unsigned grid_stream = (unsigned)sms * 4;
  k_bk_hist<<<grid_stream, BK_THREADS, 0, st>>>(q, g, hist);
  k_bk_scan<<<1, 256, 0, st>>>(hist, g, starts, cur, dcur);
  if ((e = smem_limit_raise((const void*)k_bk_scatter<true>, BK_STAGE_SMEM, dev)) ||
      (e = smem_limit_raise((const void*)k_bk_scatter<false>, BK_STAGE_SMEM, dev)) ||
      (e = smem_limit_raise((const void*)k_bk_rank<true>, BK_STAGE_SMEM, dev)) ||
      (e = smem_limit_raise((const void*)k_bk_rank<false>, BK_STAGE_SMEM, dev))) {
    cudaFreeAsync(scratch, st);
    return e;
  }
  const unsigned grid_tiles = (unsigned)sms * 2;
  if (c) {
    k_bk_scatter<true><<<grid_tiles, BK_THREADS, BK_STAGE_SMEM, st>>>(q, c, g, cur, A);
    k_bk_rank<true><<<grid_tiles, BK_THREADS, BK_STAGE_SMEM, st>>>(h->lines, h->super, A, starts, g, dcur, B, ctr);
  } else {
    k_bk_scatter<false><<<grid_tiles, BK_THREADS, BK_STAGE_SMEM, st>>>(q, c, g, cur, A);
    k_bk_rank<false><<<grid_tiles, BK_THREADS, BK_STAGE_SMEM, st>>>(h->lines, h->super, A, starts, g, dcur, B, ctr);
  }
  k_bk_unpermute<<<(unsigned)sms * 4, BK_THREADS, 0, st>>>(B, g, out, ctr + 1);
  e = cudaGetLastError();
  cudaError_t e2 = cudaFreeAsync(scratch, st);
  return e ? e : e2;
}

// BiRank16 rank through the bucketed passes; batches of more than 2^31 queries in chunks.
cudaError_t launch_bucket_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                               cudaStream_t st) {
  const uint64_t CH = g_rank_bucket_chunk;
  for (uint64_t o = 0; o < m; o += CH) {
    const uint64_t mm = m - o < CH ? m - o : CH;
    cudaError_t e = bk_chunk(h, q + o, c ? c + o : nullptr, out + o, mm, st);
    if (e) return e;
  }
  return cudaSuccess;
}

}  // namespace qr
