// sbcache.cu — rank kernels that read the superblock words from distributed shared memory.
//
// Why: on B200 a random query on an HBM-resident layout costs L2 *requests*, not bytes (DESIGN.md
// §6): the lane-pair kernels issue one request for the 64-B line, plus one for the superblock
// word s_{j>>7} / s_{j>>8,c}.  That second request is an L2 hit,
// yet it takes the same miss-path slot in the SM and costs ~16% (gather ceiling with vs without
// it, profiles/r01_s_probe.jsonl).  Here the superblock array is held in the shared memory of a
// 2-CTA cluster (one CTA per SM, 1024 threads) for the whole launch, so the only global request
// of a query is its line.
//
// The array is re-encoded losslessly so that it fits two CTAs' shared memory at the BASELINE
// sizes (n = 2^34 bits: 270,601 superblocks; n = 2^32 chars: 74,899 x 4):
//   BiRank16  — one u64 per group of 6 superblocks: bits [0,24) = s_{6g}; byte k (k = 1..5) at
//               bits [16+8k, 24+8k) = s_{6g+k} - s_{6g} <= 5*31 = 155 (each superblock adds at
//               most 128*496/2^11 = 31 to s).  Needs s < 2^24, i.e. n < 2^35.
//   QuadRank16 — per group of 8 superblocks and per symbol c one u64: bits [0,22) = s_{8g,c};
//               6-bit field k (k = 1..7) at bits [16+6k, 22+6k) = s_{8g+k,c} - s_{8g,c} <= 7*7
//               (each superblock adds at most 256*224/2^13 = 7).  Needs s < 2^22, i.e. n < 2^35.
// Group g lives in CTA (g & 1) of the cluster at local slot g >> 1; in global memory the packed
// table is stored CTA-major (slots of CTA 0, then of CTA 1) so that each CTA preloads one
// contiguous range.  The per-query arithmetic (Eq. 1, Listing 1) is unchanged: see birank.cu /
// quadrank.cu — only where s comes from differs.
#include <cooperative_groups.h>

#include <map>
#include <mutex>
#include <tuple>

#include "qr_common.cuh"
#include "sched.cuh"

namespace qr {


// ------------------------------------------------------------------ packing (build time)

__global__ void k_bi_pack_super(const uint32_t* __restrict__ super, uint64_t n_super, uint64_t groups, uint64_t half,
                                uint64_t* __restrict__ pack) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = 6 * g;
    const uint32_t s0 = super[i0];
    uint64_t w = s0;
#pragma unroll
    for (int k = 1; k < 6; ++k)
      if (i0 + k < n_super) w |= (uint64_t)(super[i0 + k] - s0) << (16 + 8 * k);
    pack[(g & 1) * half + (g >> 1)] = w;
  }
}

__global__ void k_qd_pack_super(const uint32_t* __restrict__ super, uint64_t n_super, uint64_t groups, uint64_t half,
                                uint64_t* __restrict__ pack) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < 4 * groups; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = t >> 2;
    const uint32_t c = (uint32_t)(t & 3);
    const uint64_t i0 = 8 * g;
    const uint32_t s0 = super[4 * i0 + c];
    uint64_t w = s0;
#pragma unroll
    for (int k = 1; k < 8; ++k)
      if (i0 + k < n_super) w |= (uint64_t)(super[4 * (i0 + k) + c] - s0) << (16 + 6 * k);
    pack[4 * ((g & 1) * half + (g >> 1)) + c] = w;
  }
}

static int max_dyn_smem(int device) {
  static std::mutex mu;
  static int cache[64] = {};
  std::lock_guard<std::mutex> g(mu);
  if (device < 0 || device >= 64) return 0;
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess || v <= 0) v = 1;
    cache[device] = v;
  }
  return cache[device];
}

// Bytes of shared memory one CTA of the cluster needs, or 0 when the layout cannot use the cache.
uint64_t super_pack_cta_bytes(const qr_index* h) {
  if (!h->spack) return 0;
  return h->spack_half * (h->sigma == 2 ? 8 : 32);
}

// Build h->spack from h->super (stream-ordered).  Leaves spack null (no error) when the layout
// is outside the encoding's range or the half table exceeds a CTA's shared memory.
qr_status build_super_pack_big(qr_index* h, cudaStream_t st);

qr_status build_super_pack(qr_index* h, cudaStream_t st) {
  h->spack = nullptr;
  h->spack_half = 0;
  if (qr_status sb = build_super_pack_big(h, st)) return sb;
  if (h->layout != QR_LAYOUT_BIRANK16 && h->layout != QR_LAYOUT_QUADRANK16 && h->layout != QR_LAYOUT_BIRANK16X2 &&
      h->layout != QR_LAYOUT_QUADRANK16X2)
    return QR_OK;
  if (h->n >= (1ull << 35) || h->n_super == 0) return QR_OK;     // anchors: 24 / 22 bits
  const bool bi = h->sigma == 2;
  const uint64_t groups = bi ? (h->n_super + 5) / 6 : (h->n_super + 7) / 8;
  // slots per CTA; even for BiRank so that CTA 1's range starts 16-B aligned
  const uint64_t half = bi ? (((groups + 1) / 2 + 1) & ~1ull) : (groups + 1) / 2;
  const uint64_t cta_bytes = half * (bi ? 8 : 32);
  if (cta_bytes + 1024 > (uint64_t)max_dyn_smem(h->device)) return QR_OK;
  cudaError_t e = cudaMalloc((void**)&h->spack, 2 * cta_bytes);
  if (e) { h->spack = nullptr; return cuda_fail(e, "alloc packed superblocks"); }
  cudaMemsetAsync(h->spack, 0, 2 * cta_bytes, st);
  const unsigned g = grid_stride_blocks(bi ? groups : 4 * groups, 256, h->sm_count, 8);
  if (bi) k_bi_pack_super<<<g, 256, 0, st>>>(h->super, h->n_super, groups, half, h->spack);
  else    k_qd_pack_super<<<g, 256, 0, st>>>(h->super, h->n_super, groups, half, h->spack);
  if ((e = cudaGetLastError())) { cudaFree(h->spack); h->spack = nullptr; return cuda_fail(e, "pack superblocks"); }
  h->spack_half = half;
  return QR_OK;
}

// ------------------------------------------------------------------ BiRank16 beyond 2^35 bits
// The 2-CTA table above needs s < 2^24 (n < 2^35) and half of it must fit one CTA (n <= ~2^34.4).
// For larger bit vectors (the paper's own 4 GiB, is n = 2^35) the same 6-superblock
// groups go to a wider cluster (group g at CTA g % CS, slot g / CS; CS = 4, 8 or 16), with only
// the low 24 bits of each group's base stored: bits 24-25 come from the first groups whose base
// reaches 2^24, 2^25, 3 * 2^24 (s is non-decreasing), kernel parameters — n < 2^37 bits.
__global__ void k_bi_pack_super6cs(const uint32_t* __restrict__ super, uint64_t n_super, uint64_t groups,
                                   uint64_t slots, uint32_t cs_log, uint64_t* __restrict__ pack,
                                   uint32_t* __restrict__ hi_first) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = 6 * g;
    const uint32_t s0 = super[i0];
    uint64_t w = s0 & 0xffffffu;
#pragma unroll
    for (int k = 1; k < 6; ++k)
      if (i0 + k < n_super) w |= (uint64_t)(super[i0 + k] - s0) << (16 + 8 * k);
    pack[(g & ((1ull << cs_log) - 1)) * slots + (g >> cs_log)] = w;
    // s is non-decreasing: group g is the first of high part h when its predecessor's is lower
    const uint32_t h = s0 >> 24, hp = g ? super[i0 - 6] >> 24 : 0u;
    for (uint32_t k = hp + 1; k <= h && k <= 3; ++k) hi_first[k - 1] = (uint32_t)g;
  }
}

// QuadRank16 8-superblock groups (the 2-CTA encoding) placed at CTA g % CS, slot g / CS
__global__ void k_qd_pack_super_cs(const uint32_t* __restrict__ super, uint64_t n_super, uint64_t groups,
                                   uint64_t slots, uint32_t cs_log, uint64_t* __restrict__ pack) {
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < 4 * groups; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = t >> 2;
    const uint32_t c = (uint32_t)(t & 3);
    const uint64_t i0 = 8 * g;
    const uint32_t s0 = super[4 * i0 + c];
    uint64_t w = s0;
#pragma unroll
    for (int k = 1; k < 8; ++k)
      if (i0 + k < n_super) w |= (uint64_t)(super[4 * (i0 + k) + c] - s0) << (16 + 6 * k);
    pack[4 * ((g & ((1ull << cs_log) - 1)) * slots + (g >> cs_log)) + c] = w;
  }
}

extern int g_rank_big_pack;
extern int g_rank_big_cs;

qr_status build_super_pack_big(qr_index* h, cudaStream_t st) {
  h->spack_big = nullptr;
  h->spack_big_slots = 0;
  h->spack_big_cs = 0;
  if (h->n_super == 0) return QR_OK;
  if (h->layout == QR_LAYOUT_QUADRANK16) {
    // 8-superblock groups of 32 B (22-bit base: n < 2^35 chars), for n whose 2-CTA table does
    // not fit one CTA per half (n > ~2^32.6), or forced (tests); parts <= 184 KB as for BiRank16
    // (2^34 chars: 8 x 150 KB, 40.0 Gq/s vs 37.0 at 16 x 75 KB, profiles/r01_big_qd_probe_184k.jsonl)
    if (h->n >= (1ull << 35)) return QR_OK;
    const uint64_t groups = (h->n_super + 7) / 8;
    const uint64_t half = (groups + 1) / 2;
    // also where the 2-CTA table would hold more than 184 KB per CTA: near its capacity it
    // loses to this one (n = 1.45 x 2^32: 36.6 vs 42.5 Gq/s, profiles/r01_boundary_probe.jsonl)
    if (!g_rank_big_pack && half * 32 <= 184 * 1024) return QR_OK;
    constexpr uint64_t PART_MAX = 184 * 1024;
    uint32_t cs = 0;
    for (uint32_t c = 4; c <= 16; c *= 2) {
      const uint64_t slots = (groups + c - 1) / c;
      const bool fits = slots * 32 + 1024 <= (uint64_t)max_dyn_smem(h->device);
      if (g_rank_big_cs ? (c == (uint32_t)g_rank_big_cs && fits) : (fits && slots * 32 <= PART_MAX)) { cs = c; break; }
    }
    if (!cs) return QR_OK;
    const uint32_t cs_log = cs == 4 ? 2 : cs == 8 ? 3 : 4;
    const uint64_t slots = (groups + cs - 1) / cs;
    cudaError_t e = cudaMalloc((void**)&h->spack_big, cs * slots * 32);
    if (e) { h->spack_big = nullptr; return cuda_fail(e, "alloc large superblock table"); }
    cudaMemsetAsync(h->spack_big, 0, cs * slots * 32, st);
    k_qd_pack_super_cs<<<grid_stride_blocks(4 * groups, 256, h->sm_count, 8), 256, 0, st>>>(
        h->super, h->n_super, groups, slots, cs_log, h->spack_big);
    if ((e = cudaGetLastError())) { cudaFree(h->spack_big); h->spack_big = nullptr; return cuda_fail(e, "pack superblocks"); }
    h->spack_big_slots = slots;
    h->spack_big_cs = cs;
    return QR_OK;
  }
  if (h->layout != QR_LAYOUT_BIRANK16) return QR_OK;
  if (h->n >= (1ull << 37)) return QR_OK;                            // s < 2^26: 2 high bits
  {
    // n >= 2^35 (no 2-CTA table), or a 2-CTA table of more than 184 KB per CTA (n > ~2^34.06:
    // 1.23 x 2^34 runs 34.2 Gq/s with it vs 44.1 with this one, profiles/r01_boundary_probe.jsonl)
    const uint64_t g6 = (h->n_super + 5) / 6, half6 = (((g6 + 1) / 2 + 1) & ~1ull) * 8;
    if (h->n < (1ull << 35) && half6 <= 184 * 1024 && !g_rank_big_pack) return QR_OK;
  }
  // the 2-CTA encoding (6 superblocks per u64, 24-bit base) with the base's bits 24-25 recovered
  // from three group boundaries (s is non-decreasing), split over the smallest cluster whose
  // per-CTA part is <= 184 KB — the 2-CTA table's own size at 2^34, where the kernel reaches the
  // gather ceiling; larger parts leave the L1 too little room for the misses in flight (a 216 KB
  // part: 35.4 vs 42.5 Gq/s at 108 KB, profiles/r01_big_cs_probe.jsonl)
  const uint64_t groups = (h->n_super + 5) / 6;
  const uint64_t cap = (uint64_t)max_dyn_smem(h->device);
  constexpr uint64_t PART_MAX = 184 * 1024;
  uint32_t cs = 0;
  for (uint32_t c = 4; c <= 16; c *= 2) {
    const uint64_t slots = (((groups + c - 1) / c) + 1) & ~1ull;      // even: 16-B copies
    const bool fits = slots * 8 + 1024 <= cap;
    if (g_rank_big_cs ? (c == (uint32_t)g_rank_big_cs && fits) : (fits && slots * 8 <= PART_MAX)) { cs = c; break; }
  }
  if (!cs) return QR_OK;
  const uint32_t cs_log = cs == 4 ? 2 : cs == 8 ? 3 : 4;
  const uint64_t slots = (((groups + cs - 1) / cs) + 1) & ~1ull;
  cudaError_t e = cudaMalloc((void**)&h->spack_big, cs * slots * 8 + 16);
  if (e) { h->spack_big = nullptr; return cuda_fail(e, "alloc large superblock table"); }
  uint32_t* hi_first = reinterpret_cast<uint32_t*>(h->spack_big + cs * slots);
  cudaMemsetAsync(h->spack_big, 0, cs * slots * 8, st);
  cudaMemsetAsync(hi_first, 0xff, 16, st);                             // "never": UINT32_MAX
  k_bi_pack_super6cs<<<grid_stride_blocks(groups, 256, h->sm_count, 8), 256, 0, st>>>(h->super, h->n_super, groups,
                                                                                      slots, cs_log, h->spack_big,
                                                                                      hi_first);
  if ((e = cudaGetLastError()) || (e = cudaMemcpyAsync(h->spack_big_hi, hi_first, 12, cudaMemcpyDeviceToHost, st)) ||
      (e = cudaStreamSynchronize(st))) {
    cudaFree(h->spack_big); h->spack_big = nullptr; return cuda_fail(e, "pack superblocks");
  }
  h->spack_big_slots = slots;
  h->spack_big_cs = cs;
  return QR_OK;
}

// ------------------------------------------------------------------ cluster helpers

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint64_t ld_dsmem_u64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void ld_dsmem_v2u64(uint32_t addr, uint64_t& a, uint64_t& b) {
  asm volatile("ld.shared::cluster.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}

// Preload this CTA's half of the packed table (contiguous, 16-B aligned, even word count) and make both halves
// visible cluster-wide.  Returns the shared::cluster addresses of slot 0 in CTA 0 and CTA 1.
__device__ __forceinline__ void sc_preload(const uint64_t* __restrict__ pack, uint64_t half_words, uint64_t* smem,
                                           uint32_t& base0, uint32_t& base1) {
  const uint32_t r = cluster_rank();
  const uint4* src = reinterpret_cast<const uint4*>(pack + r * half_words);
  uint4* dst = reinterpret_cast<uint4*>(smem);
  for (uint32_t i = threadIdx.x; i < (uint32_t)(half_words >> 1); i += blockDim.x) dst[i] = __ldg(src + i);
  const uint32_t local = (uint32_t)__cvta_generic_to_shared(smem);
  base0 = map_to_rank(local, 0);
  base1 = map_to_rank(local, 1);
  cluster_barrier();
}

// s_i of BiRank16 superblock i from the packed table.
__device__ __forceinline__ uint32_t bi_s_from_pack(uint32_t sb, uint32_t base0, uint32_t base1) {
  const uint32_t g = sb / 6u, k = sb - 6u * g;
  const uint64_t v = ld_dsmem_u64(((g & 1u) ? base1 : base0) + (g >> 1) * 8u);
  const uint32_t lo = (uint32_t)v & 0xffffffu;
  return k ? lo + ((uint32_t)(v >> (16u + 8u * k)) & 0xffu) : lo;
}
__device__ __forceinline__ uint32_t qd_s_field(uint64_t v, uint32_t k) {
  const uint32_t lo = (uint32_t)v & 0x3fffffu;
  return k ? lo + ((uint32_t)(v >> (16u + 6u * k)) & 0x3fu) : lo;
}

// ------------------------------------------------------------------ BiRank16 rank (Eq. 1)
// Same lane-pair structure as k_bi_rank2 (birank.cu), q < 2^36 index math; lane 1 of the pair
// reads s from the cluster's shared memory.
template <int K>
__device__ __forceinline__ void sc_load_q(const uint64_t* __restrict__ q, uint64_t i0, uint64_t step, uint64_t m,
                                          uint64_t (&qn)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint64_t idx = i0 + (uint64_t)k * step;
    qn[k] = idx < m ? ld_stream_u64(q + idx) : 0;
  }
}

// VAR bit 0: no superblock read (the shape's own gather ceiling, qr_gather_ceiling mode 3);
// VAR bit 1: dynamic work order.
template <int K, int THREADS, bool HAS_C, int VAR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_bi_rank2c(const uint4* __restrict__ lines, const uint64_t* __restrict__ pack, uint64_t half_words,
                const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                uint64_t last_line, unsigned long long* ctr) {
  constexpr bool NOS = VAR & 1, DYN = (VAR & 2) != 0;
  extern __shared__ uint64_t sc_smem[];
  uint32_t base0, base1;
  sc_preload(pack, half_words, sc_smem, base0, base1);
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = (threadIdx.x & 31u) >> 1;           // pair within the warp
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t qn[K];
  sc_load_q<K>(q, sc.gb + pw, sc.stride, m, qn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + pw;
    uint64_t qq[K];
    uint32_t jj[K], pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      qq[k] = qn[k];
      uint32_t j = (uint32_t)(qq[k] >> 4) / 31u;                // floor(q/496), q < 2^36
      j = j > (uint32_t)last_line ? (uint32_t)last_line : j;     // q > n: memory-safe clamp
      const uint64_t p = 16 + qq[k] - (uint64_t)j * BI_B;
      pp[k] = p > 511 ? 511u : (uint32_t)p;
      jj[k] = j;
    }
    uint64_t w[K][4];
    uint32_t s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (half == 0 || pp[k] >= 256) ld_sector_na(lines + 4 * (uint64_t)jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      s[k] = (half && !NOS) ? bi_s_from_pack(jj[k] >> BI_SB_LOG, base0, base1) : 0u;
    }
    const uint64_t stride = sc.stride;
    sc = sc_next<K, DYN, 16>(sc, ctr);
    sc_load_q<K>(q, sc.gb + pw, sc.stride, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      const bool right = pp[k] >= 256;
      const int x = (int)(pp[k] & 255u);
      const bool mine = half ? right : !right;
      const uint64_t inv = half ? 0ull : ~0ull;
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) cnt += __popcll(w[k][t] & (prefix_mask(x, t) ^ inv));
      cnt = mine ? cnt : 0u;
      uint64_t v = (half ? (uint64_t)cnt : (w[k][0] & 0xffffull) - cnt) + ((uint64_t)s[k] << BI_SHIFT);
      if (NOS) v = w[k][0] ^ w[k][1] ^ w[k][2] ^ w[k][3];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (HAS_C) {
        if (half == 0 && idx < m && cs[idx] == 0) v = qq[k] - v;
      }
      if (half == 0 && idx < m) st_stream_u64(out + idx, v);
    }
  }
  cluster_barrier();   // the peer may still read this CTA's half of the table
}

// BiRank16 rank over the CS-CTA table (n >= 2^35): the k_bi_rank2c structure with 64-bit line
// indices and lane 1 of a pair reading s from the CTA g % CS of its cluster.  Kept as its own body:
// sharing k_bi_rank2c's through a table policy spilled 40 B per thread here and cost 8-9%.
template <int K, int THREADS, bool HAS_C>
__global__ void __launch_bounds__(THREADS, 1)
    k_bi_rank2v(const uint4* __restrict__ lines, const uint64_t* __restrict__ pack, uint64_t slots, uint32_t cs_log, uint32_t hi1, uint32_t hi2,
                uint32_t hi3,
                const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                uint64_t last_line, unsigned long long* ctr) {
  extern __shared__ uint64_t sc_smem[];
  {
    const uint4* src = reinterpret_cast<const uint4*>(pack + (uint64_t)cluster_rank() * slots);
    uint4* dst = reinterpret_cast<uint4*>(sc_smem);
    for (uint32_t i = threadIdx.x; i < (uint32_t)(slots >> 1); i += blockDim.x) dst[i] = __ldg(src + i);
    cluster_barrier();
  }
  const uint32_t local = (uint32_t)__cvta_generic_to_shared(sc_smem);
  const uint32_t csm = (1u << cs_log) - 1u;
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = (threadIdx.x & 31u) >> 1;
  ScSched sc = sc_first<K, true, 16>(ctr);
  uint64_t qn[K];
  sc_load_q<K>(q, sc.gb + pw, sc.stride, m, qn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + pw;
    uint64_t qq[K], jj[K];
    uint32_t pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      qq[k] = qn[k];
      uint64_t j = qq[k] / BI_B;
      j = j > last_line ? last_line : j;                           // q > n: memory-safe clamp
      const uint64_t p = 16 + qq[k] - j * BI_B;
      pp[k] = p > 511 ? 511u : (uint32_t)p;
      jj[k] = j;
    }
    uint64_t w[K][4];
    uint32_t s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (half == 0 || pp[k] >= 256) ld_sector_na(lines + 4 * jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      s[k] = 0;
      if (half) {
        const uint32_t sb = (uint32_t)(jj[k] >> BI_SB_LOG), g = sb / 6u, kk = sb - 6u * g;
        const uint64_t v = ld_dsmem_u64(map_to_rank(local, g & csm) + (g >> cs_log) * 8u);
        const uint32_t base = ((uint32_t)v & 0xffffffu) |
                              (((uint32_t)(g >= hi1) + (uint32_t)(g >= hi2) + (uint32_t)(g >= hi3)) << 24);
        s[k] = kk ? base + ((uint32_t)(v >> (16u + 8u * kk)) & 0xffu) : base;
      }
    }
    const uint64_t stride = sc.stride;
    sc = sc_next<K, true, 16>(sc, ctr);
    sc_load_q<K>(q, sc.gb + pw, sc.stride, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      const bool right = pp[k] >= 256;
      const int x = (int)(pp[k] & 255u);
      const bool mine = half ? right : !right;
      const uint64_t inv = half ? 0ull : ~0ull;
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) cnt += __popcll(w[k][t] & (prefix_mask(x, t) ^ inv));
      cnt = mine ? cnt : 0u;
      uint64_t v = (half ? (uint64_t)cnt : (w[k][0] & 0xffffull) - cnt) + ((uint64_t)s[k] << BI_SHIFT);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (HAS_C) {
        if (half == 0 && idx < m && cs[idx] == 0) v = qq[k] - v;
      }
      if (half == 0 && idx < m) st_stream_u64(out + idx, v);
    }
  }
  cluster_barrier();   // the peers may still read this CTA's part of the table
}

// ------------------------------------------------------------------ QuadRank16 rank(q,c), rank_4(q)
template <int K, bool WITH_C>
__device__ __forceinline__ void sc_load_qc(const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs, uint64_t i0,
                                           uint64_t step, uint64_t m, uint64_t (&qn)[K], uint32_t (&cn)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint64_t idx = i0 + (uint64_t)k * step;
    qn[k] = idx < m ? ld_stream_u64(q + idx) : 0;
    if (WITH_C) cn[k] = idx < m ? ld_stream_u8(cs + idx) & 3u : 0u;
  }
}

template <int K>
__device__ __forceinline__ void qd_locate32(const uint64_t (&qq)[K], uint64_t last_line, uint32_t (&jj)[K],
                                            uint32_t (&pp)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uint32_t j = (uint32_t)(qq[k] >> 5) / 7u;                  // floor(q/224), q < 2^37
    j = j > (uint32_t)last_line ? (uint32_t)last_line : j;
    const uint64_t p = 32 + qq[k] - (uint64_t)j * QD_B;
    pp[k] = p > 255 ? 255u : (uint32_t)p;
    jj[k] = j;
  }
}

// Address of QuadRank16 group g's 32-B record in the cluster's shared memory: the 2-CTA table
// (CTA g & 1, addresses of both CTAs mapped once) or the CS-CTA table (CTA g % CS, mapa per read).
struct QdTable2 {
  uint32_t base0, base1;
  __device__ __forceinline__ uint32_t addr(uint32_t g) const { return ((g & 1u) ? base1 : base0) + (g >> 1) * 32u; }
};
struct QdTableCS {
  uint32_t local, csm, cs_log;
  __device__ __forceinline__ uint32_t addr(uint32_t g) const { return map_to_rank(local, g & csm) + (g >> cs_log) * 32u; }
};

// Bodies of the QuadRank16 cluster kernels (rank(q,c) and rank_4), shared by the 2-CTA and the
// CS-CTA entry points below.
template <int K, bool DYN, class TBL>
__device__ __forceinline__ void qd_rank2_body(const uint4* __restrict__ lines, const TBL& tbl,
                                              const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                              uint64_t* __restrict__ out, uint64_t m, uint64_t last_line,
                                              unsigned long long* ctr) {
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = (threadIdx.x & 31u) >> 1;
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t qn[K];
  uint32_t cn[K];
  sc_load_qc<K, true>(q, cs, sc.gb + pw, sc.stride, m, qn, cn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + pw;
    uint64_t qq[K];
    uint32_t jj[K], pp[K], cc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { qq[k] = qn[k]; cc[k] = cn[k]; }
    qd_locate32<K>(qq, last_line, jj, pp);
    uint64_t w[K][4];
    uint32_t s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (half == 0 || pp[k] >= 128) ld_sector_na(lines + 4 * (uint64_t)jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      s[k] = 0;
      if (half) {
        const uint32_t sb = jj[k] >> QD_SB_LOG, g = sb >> 3;
        s[k] = qd_s_field(ld_dsmem_u64(tbl.addr(g) + 8u * cc[k]), sb & 7u);
      }
    }
    const uint64_t stride = sc.stride;
    sc = sc_next<K, DYN, 16>(sc, ctr);
    sc_load_qc<K, true>(q, cs, sc.gb + pw, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      const bool right = pp[k] >= 128;
      const bool mine = half ? right : !right;
      const uint64_t cl = 0ull - (uint64_t)(cc[k] & 1u), ch = 0ull - (uint64_t)(cc[k] >> 1);
      const int x = (int)(pp[k] & 127u);
      const uint64_t inv = half ? 0ull : ~0ull;
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) cnt += __popcll((w[k][2 * t] ^ cl) & (w[k][2 * t + 1] ^ ch) & (prefix_mask(x, t) ^ inv));
      cnt = mine ? cnt : 0u;
      const uint64_t dw = (cc[k] & 2u) ? w[k][1] : w[k][0];
      const uint64_t delta = (dw >> (16 * (cc[k] & 1u))) & 0xffffull;      // u16 slot c + (c & 2)
      uint64_t v = (half ? (uint64_t)cnt : delta - cnt) + ((uint64_t)s[k] << QD_SHIFT);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (half == 0 && idx < m) st_stream_u64(out + idx, v);
    }
  }
}

template <int K, bool DYN, class TBL>
__device__ __forceinline__ void qd_all4_2_body(const uint4* __restrict__ lines, const TBL& tbl,
                                               const uint64_t* __restrict__ q, uint64_t* __restrict__ out4, uint64_t m,
                                               uint64_t last_line, unsigned long long* ctr) {
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t pw = (threadIdx.x & 31u) >> 1;
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t qn[K];
  uint32_t cn[K];
  sc_load_qc<K, false>(q, nullptr, sc.gb + pw, sc.stride, m, qn, cn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + pw;
    uint64_t qq[K];
    uint32_t jj[K], pp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) qq[k] = qn[k];
    qd_locate32<K>(qq, last_line, jj, pp);
    uint64_t w[K][4];
    uint32_t s0[K], s1[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0;
      if (half == 0 || pp[k] >= 128) ld_sector_na(lines + 4 * (uint64_t)jj[k] + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      // lane 0: s_A, s_C; lane 1: s_G, s_T (adjacent u64 fields of the group)
      const uint32_t sb = jj[k] >> QD_SB_LOG, g = sb >> 3;
      uint64_t va, vb;
      ld_dsmem_v2u64(tbl.addr(g) + 16u * half, va, vb);
      s0[k] = qd_s_field(va, sb & 7u);
      s1[k] = qd_s_field(vb, sb & 7u);
    }
    const uint64_t stride = sc.stride;
    sc = sc_next<K, DYN, 16>(sc, ctr);
    sc_load_qc<K, false>(q, nullptr, sc.gb + pw, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      const bool right = pp[k] >= 128;
      const int x = (int)(pp[k] & 127u);
      const uint64_t inv = half ? 0ull : ~0ull;
      uint32_t nl = 0, nh = 0, nt = 0;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const uint64_t msk = prefix_mask(x, t) ^ inv;
        const uint64_t l = ~w[k][2 * t] & msk, hh = ~w[k][2 * t + 1] & msk;   // planes store the negation
        nl += __popcll(l);
        nh += __popcll(hh);
        nt += __popcll(l & hh);
      }
      const uint32_t len = half ? (uint32_t)x : 128u - (uint32_t)x;
      const uint32_t packed = (len - nl - nh + nt) | ((nl - nt) << 8) | ((nh - nt) << 16) | (nt << 24);
      const uint32_t other = __shfl_xor_sync(0xffffffffu, packed, 1);
      const uint32_t dgt = __shfl_xor_sync(0xffffffffu, (uint32_t)w[k][1], 1);
      const uint32_t cnt = (right == (half == 1)) ? packed : other;
      const uint32_t dl = half ? dgt : (uint32_t)w[k][0];
      const uint32_t c0 = (cnt >> (16 * half)) & 0xffu, c1 = (cnt >> (16 * half + 8)) & 0xffu;
      const uint64_t b0 = ((uint64_t)s0[k] << QD_SHIFT) + (dl & 0xffffu);
      const uint64_t b1 = ((uint64_t)s1[k] << QD_SHIFT) + (dl >> 16);
      const uint64_t r0 = right ? b0 + c0 : b0 - c0, r1 = right ? b1 + c1 : b1 - c1;
      if (idx < m) asm volatile("st.global.L1::no_allocate.v2.u64 [%0], {%1,%2};" ::"l"(out4 + 4 * idx + 2 * half),
                                "l"(r0), "l"(r1) : "memory");
    }
  }
}

template <int K, int THREADS, bool DYN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_qd_rank2c(const uint4* __restrict__ lines, const uint64_t* __restrict__ pack, uint64_t half_words,
                const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                uint64_t last_line, unsigned long long* ctr) {
  extern __shared__ uint64_t sc_smem[];
  uint32_t base0, base1;
  sc_preload(pack, half_words, sc_smem, base0, base1);
  qd_rank2_body<K, DYN>(lines, QdTable2{base0, base1}, q, cs, out, m, last_line, ctr);
  cluster_barrier();
}

template <int K, int THREADS, bool DYN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_qd_all4_2c(const uint4* __restrict__ lines, const uint64_t* __restrict__ pack, uint64_t half_words,
                 const uint64_t* __restrict__ q, uint64_t* __restrict__ out4, uint64_t m, uint64_t last_line,
                 unsigned long long* ctr) {
  extern __shared__ uint64_t sc_smem[];
  uint32_t base0, base1;
  sc_preload(pack, half_words, sc_smem, base0, base1);
  qd_all4_2_body<K, DYN>(lines, QdTable2{base0, base1}, q, out4, m, last_line, ctr);
  cluster_barrier();
}

// QuadRank16 rank / rank_4 over a CS-CTA cluster table (n > ~2^32.6 chars, where half the
// 2-CTA table no longer fits one CTA; the paper's 4 GiB text is n = 2^34): the k_qd_rank2c /
// k_qd_all4_2c bodies with the same 8-superblock groups (22-bit base: n < 2^35) placed at CTA
// g % CS, slot g / CS, and the dynamic work order.
template <int K, int THREADS>
__global__ void __launch_bounds__(THREADS, 1)
    k_qd_rank2w(const uint4* __restrict__ lines, const uint64_t* __restrict__ pack, uint64_t part_words, uint32_t cs_log,
                const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                uint64_t last_line, unsigned long long* ctr) {
  extern __shared__ uint64_t sc_smem[];
  {
    const uint4* src = reinterpret_cast<const uint4*>(pack + (uint64_t)cluster_rank() * part_words);
    uint4* dst = reinterpret_cast<uint4*>(sc_smem);
    for (uint32_t i = threadIdx.x; i < (uint32_t)(part_words >> 1); i += blockDim.x) dst[i] = __ldg(src + i);
    cluster_barrier();
  }
  const uint32_t local = (uint32_t)__cvta_generic_to_shared(sc_smem);
  const uint32_t csm = (1u << cs_log) - 1u;
  qd_rank2_body<K, true>(lines, QdTableCS{local, csm, cs_log}, q, cs, out, m, last_line, ctr);
  cluster_barrier();
}


template <int K, int THREADS>
__global__ void __launch_bounds__(THREADS, 1)
    k_qd_all4_2w(const uint4* __restrict__ lines, const uint64_t* __restrict__ pack, uint64_t part_words, uint32_t cs_log,
                 const uint64_t* __restrict__ q, uint64_t* __restrict__ out4, uint64_t m, uint64_t last_line,
                 unsigned long long* ctr) {
  extern __shared__ uint64_t sc_smem[];
  {
    const uint4* src = reinterpret_cast<const uint4*>(pack + (uint64_t)cluster_rank() * part_words);
    uint4* dst = reinterpret_cast<uint4*>(sc_smem);
    for (uint32_t i = threadIdx.x; i < (uint32_t)(part_words >> 1); i += blockDim.x) dst[i] = __ldg(src + i);
    cluster_barrier();
  }
  const uint32_t local = (uint32_t)__cvta_generic_to_shared(sc_smem);
  const uint32_t csm = (1u << cs_log) - 1u;
  qd_all4_2_body<K, true>(lines, QdTableCS{local, csm, cs_log}, q, out4, m, last_line, ctr);
  cluster_barrier();
}


// ------------------------------------------------------------------ one lane per query, table per CTA
// For L2-resident structures (rank_shape LANE) the line requests are cheap L2 hits and the cost
// is instructions: one lane per query beats lane pairs (135 vs 98 Gq/s at 33 MB, profiles/
// r01_regime_probe.jsonl).  These kernels take the superblock word from a private copy of the
// whole packed table in each CTA's shared memory (small at these sizes: <= 32 KB), so that the
// line is the query's only global request.  Line loads as in k_bi_rank / k_qd_rank: sector 0
// always, sector 1 for queries right of the anchor (the L1 merges both into one L2 request).
constexpr uint64_t LANE_TABLE_MAX = 32 * 1024;
extern int g_rank_blocks_per_sm;

__device__ __forceinline__ void lane_preload(const uint64_t* __restrict__ pack, uint32_t words, uint64_t* smem) {
  const uint4* src = reinterpret_cast<const uint4*>(pack);
  uint4* dst = reinterpret_cast<uint4*>(smem);
  for (uint32_t i = threadIdx.x; i < words / 2; i += blockDim.x) dst[i] = __ldg(src + i);
  __syncthreads();
}

// Resident variant (RES): structures whose whole line array fits next to the table in one CTA's
// shared memory (<= RES_MAX, e.g. configs[0]: 135 KB) are copied in once per CTA, and every query
// reads its line from shared memory — no L2 request per query, and no hot-spotting of the few
// L2 lines that all queries of a small structure hit (69 Gq/s at configs[0] with lines from L2).
// Returns the line array the kernel reads: global (RES = false) or its shared-memory copy.
template <bool RES>
__device__ __forceinline__ const uint4* lane_preload_lines(const uint64_t* __restrict__ pack, uint32_t words,
                                                           const uint4* __restrict__ lines, uint32_t line_u4,
                                                           uint64_t* smem) {
  if (!RES) {
    lane_preload(pack, words, smem);
    return lines;
  }
  const uint4* src = reinterpret_cast<const uint4*>(pack);
  uint4* dst = reinterpret_cast<uint4*>(smem);
  for (uint32_t i = threadIdx.x; i < words / 2; i += blockDim.x) dst[i] = __ldg(src + i);
  // 16-B chunk c of line j is stored at chunk 4j + (c ^ (j & 3)): without the swizzle every
  // line starts on bank 0 or 16, so a warp's 32 random lines pile onto 8 banks (ncu: ~28 shared
  // wavefronts per 16-B load, the kernel bound by them); with it the first chunks spread over
  // all 32 banks
  uint4* ldst = reinterpret_cast<uint4*>(smem + words);
  for (uint32_t i = threadIdx.x; i < line_u4; i += blockDim.x)
    ldst[(i & ~3u) | ((i & 3u) ^ ((i >> 2) & 3u))] = __ldg(lines + i);
  __syncthreads();
  return ldst;
}

// 32-B sector `sec` of line j: global (non-allocating L1) or the swizzled shared-memory copy
template <bool RES>
__device__ __forceinline__ void lane_sector(const uint4* lines, uint64_t j, uint32_t sec, uint64_t& w0, uint64_t& w1,
                                            uint64_t& w2, uint64_t& w3) {
  if (RES) {
    const uint32_t sw = (uint32_t)j & 3u, base = 4u * (uint32_t)j;
    const uint4 x = lines[base + ((2u * sec) ^ sw)], y = lines[base + ((2u * sec + 1u) ^ sw)];
    w0 = ((uint64_t)x.y << 32) | x.x; w1 = ((uint64_t)x.w << 32) | x.z;
    w2 = ((uint64_t)y.y << 32) | y.x; w3 = ((uint64_t)y.w << 32) | y.z;
  } else {
    ld_sector_na(lines + 4 * j + 2 * sec, w0, w1, w2, w3);
  }
}

// packed BiRank group g lives at part (g & 1), slot g >> 1 (half = slots per part)
__device__ __forceinline__ uint32_t bi_s_local(const uint64_t* smem, uint32_t half, uint32_t sb) {
  const uint32_t g = sb / 6u, k = sb - 6u * g;
  const uint64_t v = smem[(g & 1u) * half + (g >> 1)];
  const uint32_t lo = (uint32_t)v & 0xffffffu;
  return k ? lo + ((uint32_t)(v >> (16u + 8u * k)) & 0xffu) : lo;
}

template <int K, bool HAS_C, bool DYN, bool RES = false>
__global__ void __launch_bounds__(RES ? 1024 : 256) k_bi_rank1s(const uint4* __restrict__ lines_g,
                                                   const uint64_t* __restrict__ pack,
                                                   uint32_t words, uint32_t half, const uint64_t* __restrict__ q,
                                                   const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                                                   uint64_t last_line, unsigned long long* ctr) {
  extern __shared__ uint64_t lt_smem[];
  const uint4* lines = lane_preload_lines<RES>(pack, words, lines_g, RES ? 4u * (uint32_t)(last_line + 1) : 0u, lt_smem);
  const uint32_t u = sc_unit_in_warp<32>();
  ScSched sc = sc_first<K, DYN, 32>(ctr);
  uint64_t qn[K];
  sc_load_q<K>(q, sc.gb + u, sc.stride, m, qn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, stride = sc.stride;
    uint64_t qq[K], a[K][4], b[K][4];
    uint32_t jj[K], pp[K], s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      qq[k] = qn[k];
      uint32_t j = (uint32_t)(qq[k] >> 4) / 31u;                // floor(q/496), q < 2^36
      j = j > (uint32_t)last_line ? (uint32_t)last_line : j;     // q > n: memory-safe clamp
      const uint64_t p = 16 + qq[k] - (uint64_t)j * BI_B;
      pp[k] = p > 511 ? 511u : (uint32_t)p;
      jj[k] = j;
      lane_sector<RES>(lines, j, 0, a[k][0], a[k][1], a[k][2], a[k][3]);
      b[k][0] = b[k][1] = b[k][2] = b[k][3] = 0;
      if (pp[k] >= 256) lane_sector<RES>(lines, j, 1, b[k][0], b[k][1], b[k][2], b[k][3]);
      s[k] = bi_s_local(lt_smem, half, j >> BI_SB_LOG);
    }
    sc = sc_next<K, DYN, 32>(sc, ctr);
    sc_load_q<K>(q, sc.gb + u, sc.stride, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      const bool right = pp[k] >= 256;
      const int x = (int)(pp[k] & 255u);
      const uint64_t inv = right ? 0ull : ~0ull;
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) cnt += __popcll((right ? b[k][t] : a[k][t]) & (prefix_mask(x, t) ^ inv));
      const uint64_t base = ((uint64_t)s[k] << BI_SHIFT) + (a[k][0] & 0xffffull);
      uint64_t r = right ? base + cnt : base - cnt;
      if (HAS_C) {
        if (idx < m && cs[idx] == 0) r = qq[k] - r;
      }
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
}

// packed QuadRank group g: 4 u64 (one per symbol) at part (g & 1), slot g >> 1
__device__ __forceinline__ const uint64_t* qd_group_local(const uint64_t* smem, uint32_t half, uint32_t g) {
  return smem + 4 * ((g & 1u) * half + (g >> 1));
}

template <int K, int MODE, bool DYN, bool RES = false>   // MODE 0: rank(q,c); 1: rank_4(q)
__global__ void __launch_bounds__(RES ? 1024 : 256) k_qd_rank1s(const uint4* __restrict__ lines_g,
                                                   const uint64_t* __restrict__ pack,
                                                   uint32_t words, uint32_t half, const uint64_t* __restrict__ q,
                                                   const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                                                   uint64_t last_line, unsigned long long* ctr) {
  extern __shared__ uint64_t lt_smem[];
  const uint4* lines = lane_preload_lines<RES>(pack, words, lines_g, RES ? 4u * (uint32_t)(last_line + 1) : 0u, lt_smem);
  const uint32_t u = sc_unit_in_warp<32>();
  ScSched sc = sc_first<K, DYN, 32>(ctr);
  uint64_t qn[K];
  uint32_t cn[K];
  sc_load_qc<K, MODE == 0>(q, cs, sc.gb + u, sc.stride, m, qn, cn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, stride = sc.stride;
    uint64_t qq[K], a[K][4], b[K][4];
    uint32_t jj[K], pp[K], cc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { qq[k] = qn[k]; cc[k] = MODE == 0 ? cn[k] : 0u; }
    qd_locate32<K>(qq, last_line, jj, pp);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      lane_sector<RES>(lines, jj[k], 0, a[k][0], a[k][1], a[k][2], a[k][3]);
      b[k][0] = b[k][1] = b[k][2] = b[k][3] = 0;
      if (pp[k] >= 128) lane_sector<RES>(lines, jj[k], 1, b[k][0], b[k][1], b[k][2], b[k][3]);
    }
    sc = sc_next<K, DYN, 32>(sc, ctr);
    sc_load_qc<K, MODE == 0>(q, cs, sc.gb + u, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      const bool right = pp[k] >= 128;
      const int x = (int)(pp[k] & 127u);
      const uint64_t inv = right ? 0ull : ~0ull;
      const uint64_t* w = right ? b[k] : a[k];
      const uint32_t sb = jj[k] >> QD_SB_LOG, g = sb >> 3, sk = sb & 7u;
      const uint64_t* grp = qd_group_local(lt_smem, half, g);
      if (MODE == 0) {
        const uint32_t c = cc[k];
        const uint64_t cl = 0ull - (uint64_t)(c & 1u), ch = 0ull - (uint64_t)(c >> 1);
        uint32_t cnt = 0;
#pragma unroll
        for (int t = 0; t < 2; ++t) cnt += __popcll((w[2 * t] ^ cl) & (w[2 * t + 1] ^ ch) & (prefix_mask(x, t) ^ inv));
        const uint64_t dw = (c & 2u) ? a[k][1] : a[k][0];
        const uint64_t delta = (dw >> (16 * (c & 1u))) & 0xffffull;        // u16 slot c + (c & 2)
        const uint64_t base = ((uint64_t)qd_s_field(grp[c], sk) << QD_SHIFT) + delta;
        if (idx < m) st_stream_u64(out + idx, right ? base + cnt : base - cnt);
      } else {
        uint32_t nl = 0, nh = 0, nt = 0;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const uint64_t msk = prefix_mask(x, t) ^ inv;
          const uint64_t l = ~w[2 * t] & msk, hh = ~w[2 * t + 1] & msk;   // planes store the negation
          nl += __popcll(l);
          nh += __popcll(hh);
          nt += __popcll(l & hh);
        }
        const uint32_t len = right ? (uint32_t)x : 128u - (uint32_t)x;
        const uint32_t cnt[4] = {len - nl - nh + nt, nl - nt, nh - nt, nt};
        uint64_t r[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint64_t dw = (c & 2) ? a[k][1] : a[k][0];
          const uint64_t base = ((uint64_t)qd_s_field(grp[c], sk) << QD_SHIFT) + ((dw >> (16 * (c & 1))) & 0xffffull);
          r[c] = right ? base + cnt[c] : base - cnt[c];
        }
        if (idx < m) st_stream_v4u64(out + 4 * idx, r[0], r[1], r[2], r[3]);
      }
    }
  }
}

// ------------------------------------------------------------------ BiRank16x2 (one sector per query)
// Query q (variants.cu: layout): j = q / 480, d = q - 480 j, sector h = [d >= 240], x = d - 240 h;
// the sector's anchor is its data bit 120 = sector bit 136, its delta the sector's low 16 bits:
// rank = 2^11 s_{j>>7} + delta +- popc(sector bits between 16 + x and 136) (PAPER.md:484-485:
// at most 120 bits, "only a quarter of the cache line").  One lane per query, one 32-B load.
// SRC: 0 superblock word from L2, 1 from a per-CTA copy of the packed table; the cluster kernel
// below reads it from 2-CTA cluster shared memory.  MODE 1 = the gather ceiling (same load).
template <int K>
__device__ __forceinline__ void b16x2_locate(uint64_t q, uint64_t last_line, uint32_t& j, uint32_t& h, uint32_t& x) {
  uint32_t jj = q < (1ull << 37) ? (uint32_t)(q >> 5) / 15u    // floor(q/480) in 32 bits
                                 : (uint32_t)(q / B16X2_B);    // (lines < 2^32: n < 2^40)
  jj = jj > (uint32_t)last_line ? (uint32_t)last_line : jj;   // q > n: memory-safe clamp
  uint64_t d = q - (uint64_t)jj * B16X2_B;
  d = d > B16X2_B - 1 ? B16X2_B - 1 : d;
  h = d >= 240 ? 1u : 0u;
  x = (uint32_t)d - 240u * h;
  j = jj;
}

__device__ __forceinline__ uint64_t b16x2_value(const uint64_t (&w)[4], uint32_t x, uint32_t s) {
  uint32_t cnt = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) cnt += __popcll(w[t] & (prefix_mask(16 + (int)x, t) ^ prefix_mask(136, t)));
  const uint64_t base = ((uint64_t)s << BI_SHIFT) + (w[0] & 0xffffull);
  return x >= 120 ? base + cnt : base - cnt;
}

template <int K, int SRC, int MODE, bool HAS_C, bool DYN>
__global__ void __launch_bounds__(256) k_b16x2_rank(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                    const uint64_t* __restrict__ pack, uint32_t words, uint32_t half,
                                                    const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                                    uint64_t* __restrict__ out, uint64_t m, uint64_t last_line,
                                                    unsigned long long* ctr) {
  extern __shared__ uint64_t lt_smem[];
  if (SRC == 1) lane_preload(pack, words, lt_smem);
  const uint32_t u = sc_unit_in_warp<32>();
  ScSched sc = sc_first<K, DYN, 32>(ctr);
  uint64_t qn[K];
  sc_load_q<K>(q, sc.gb + u, sc.stride, m, qn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, stride = sc.stride;
    uint64_t qq[K], w[K][4];
    uint32_t xx[K], s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      qq[k] = qn[k];
      uint32_t j, h, x;
      b16x2_locate<K>(qq[k], last_line, j, h, x);
      xx[k] = x;
      ld_sector_na(lines + 4 * (uint64_t)j + 2 * h, w[k][0], w[k][1], w[k][2], w[k][3]);
      s[k] = MODE == 1 ? 0u : SRC == 1 ? bi_s_local(lt_smem, half, j >> BI_SB_LOG) : __ldg(super + (j >> BI_SB_LOG));
    }
    sc = sc_next<K, DYN, 32>(sc, ctr);
    sc_load_q<K>(q, sc.gb + u, sc.stride, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      uint64_t r = MODE == 1 ? (w[k][0] ^ w[k][1] ^ w[k][2] ^ w[k][3]) : b16x2_value(w[k], xx[k], s[k]);
      if (HAS_C && MODE == 0) {
        if (idx < m && cs[idx] == 0) r = qq[k] - r;
      }
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
}

template <int K, int THREADS, bool HAS_C, bool DYN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_b16x2_rank_c(const uint4* __restrict__ lines, const uint64_t* __restrict__ pack, uint64_t half_words,
                   const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                   uint64_t last_line, unsigned long long* ctr) {
  extern __shared__ uint64_t sc_smem[];
  uint32_t base0, base1;
  sc_preload(pack, half_words, sc_smem, base0, base1);
  const uint32_t u = sc_unit_in_warp<32>();
  ScSched sc = sc_first<K, DYN, 32>(ctr);
  uint64_t qn[K];
  sc_load_q<K>(q, sc.gb + u, sc.stride, m, qn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, stride = sc.stride;
    uint64_t qq[K], w[K][4];
    uint32_t xx[K], s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      qq[k] = qn[k];
      uint32_t j, h, x;
      b16x2_locate<K>(qq[k], last_line, j, h, x);
      xx[k] = x;
      ld_sector_na(lines + 4 * (uint64_t)j + 2 * h, w[k][0], w[k][1], w[k][2], w[k][3]);
      s[k] = bi_s_from_pack(j >> BI_SB_LOG, base0, base1);
    }
    sc = sc_next<K, DYN, 32>(sc, ctr);
    sc_load_q<K>(q, sc.gb + u, sc.stride, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      uint64_t r = b16x2_value(w[k], xx[k], s[k]);
      if (HAS_C) {
        if (idx < m && cs[idx] == 0) r = qq[k] - r;
      }
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
  cluster_barrier();
}

// ------------------------------------------------------------------ BiRank32x2 (one sector per query)
// Query: j = q / 448, d = q - 448 j, sector h = [d >= 224], x = d - 224 h; the sector's u32 delta
// is relative to L1[j >> 23], its anchor is data bit 112 = sector bit 144:
// rank = L1 + delta +- popc(sector bits between 32 + x and 144).  The whole L1 array is copied
// into each CTA's shared memory (<= 18.7 KB for any n < 2^43), so a query's only global load is
// its sector.  MODE 1: gather ceiling (same load).
template <int K, int MODE, bool HAS_C, bool DYN>
__global__ void __launch_bounds__(256) k_b32x2_rank(const uint4* __restrict__ lines, const uint64_t* __restrict__ l1,
                                                    uint32_t l1_words, const uint64_t* __restrict__ q,
                                                    const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                                                    uint64_t last_line, unsigned long long* ctr) {
  extern __shared__ uint64_t lt_smem[];
  for (uint32_t i = threadIdx.x; i < l1_words; i += blockDim.x) lt_smem[i] = __ldg(l1 + i);
  __syncthreads();
  const uint32_t u = sc_unit_in_warp<32>();
  ScSched sc = sc_first<K, DYN, 32>(ctr);
  uint64_t qn[K];
  sc_load_q<K>(q, sc.gb + u, sc.stride, m, qn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, stride = sc.stride;
    uint64_t qq[K], w[K][4], base[K];
    uint32_t xx[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      qq[k] = qn[k];
      uint64_t j = qq[k] < (1ull << 37) ? (uint64_t)((uint32_t)(qq[k] >> 6) / 7u) : qq[k] / B32X2_B;   // floor(q/448)
      j = j > last_line ? last_line : j;
      uint64_t d = qq[k] - j * B32X2_B;
      d = d > B32X2_B - 1 ? B32X2_B - 1 : d;
      const uint32_t h = d >= 224 ? 1u : 0u;
      xx[k] = (uint32_t)d - 224u * h;
      ld_sector_na(lines + 4 * j + 2 * h, w[k][0], w[k][1], w[k][2], w[k][3]);
      base[k] = MODE == 1 ? 0ull : lt_smem[j >> B32X2_SB_LOG];
    }
    sc = sc_next<K, DYN, 32>(sc, ctr);
    sc_load_q<K>(q, sc.gb + u, sc.stride, m, qn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      uint64_t r;
      if (MODE == 1) {
        r = w[k][0] ^ w[k][1] ^ w[k][2] ^ w[k][3];
      } else {
        uint32_t cnt = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) cnt += __popcll(w[k][t] & (prefix_mask(32 + (int)xx[k], t) ^ prefix_mask(144, t)));
        const uint64_t b = base[k] + (w[k][0] & 0xffffffffull);
        r = xx[k] >= 112 ? b + cnt : b - cnt;
        if (HAS_C) {
          if (idx < m && cs[idx] == 0) r = qq[k] - r;
        }
      }
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
}

// ------------------------------------------------------------------ QuadRank16x2 (one sector per query)
// Query (variants.cu: layout): j = q / 192, d = q - 192 j, sector h = [d >= 96], x = d - 96 h;
// anchor = the sector's char 48; its word 0 holds the four u16 deltas (c at bits 16 c), words
// 1..3 the 96 chars as transposed bit planes (variants.cu).  rank(q,c) = 2^13 s_{j>>8,c} + d_c +- #c in the chars
// between x and 48 (<= 48 chars); rank_4 from three plane popcounts (A = len - L - H + T).
__device__ __forceinline__ void q16x2_locate(uint64_t q, uint64_t last_line, uint32_t& j, uint32_t& h, uint32_t& x) {
  uint32_t jj = q < (1ull << 38) ? (uint32_t)(q >> 6) / 3u : (uint32_t)(q / Q16X2_B);   // floor(q/192)
  jj = jj > (uint32_t)last_line ? (uint32_t)last_line : jj;
  uint64_t d = q - (uint64_t)jj * Q16X2_B;
  d = d > Q16X2_B - 1 ? Q16X2_B - 1 : d;
  h = d >= 96 ? 1u : 0u;
  x = (uint32_t)d - 96u * h;
  j = jj;
}

// mask of the chars between x and 48 (symmetric difference of two prefixes) in plane word t
// (t = 0: chars 0..63; t = 1: chars 64..95 in the low 32 bits)
__device__ __forceinline__ uint64_t q16x2_range(uint32_t x, int t) {
  return (prefix_mask((int)x, t) ^ prefix_mask(48, t)) & (t ? 0xffffffffull : ~0ull);
}

__device__ __forceinline__ uint64_t q16x2_rank1(const uint64_t (&w)[4], uint32_t x, uint32_t c, uint32_t s) {
  const uint64_t nl = (c & 1u) ? 0ull : ~0ull, nh = (c & 2u) ? 0ull : ~0ull;
  const uint32_t cnt = __popcll((w[1] ^ nl) & (w[2] ^ nh) & q16x2_range(x, 0)) +
                       __popcll((w[3] ^ nl) & ((w[3] >> 32) ^ nh) & q16x2_range(x, 1));
  const uint64_t base = ((uint64_t)s << QD_SHIFT) + ((w[0] >> (16 * c)) & 0xffffull);
  return x >= 48 ? base + cnt : base - cnt;
}

__device__ __forceinline__ void q16x2_rank4(const uint64_t (&w)[4], uint32_t x, const uint32_t (&s)[4], uint64_t (&r)[4]) {
  const uint64_t m0 = q16x2_range(x, 0), m1 = q16x2_range(x, 1);
  const uint64_t l0 = w[1] & m0, h0 = w[2] & m0, l1 = w[3] & m1, h1 = (w[3] >> 32) & m1;
  const uint32_t nl = __popcll(l0) + __popcll(l1), nh = __popcll(h0) + __popcll(h1);
  const uint32_t nt = __popcll(l0 & h0) + __popcll(l1 & h1);
  const uint32_t len = x >= 48 ? x - 48u : 48u - x;
  const uint32_t cnt[4] = {len - nl - nh + nt, nl - nt, nh - nt, nt};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint64_t base = ((uint64_t)s[c] << QD_SHIFT) + ((w[0] >> (16 * c)) & 0xffffull);
    r[c] = x >= 48 ? base + cnt[c] : base - cnt[c];
  }
}

template <int K, int SRC, int MODE, bool DYN>   // SRC 0: s from L2, 1: per-CTA table; MODE 0 rank, 1 rank_4, 2 gather
__global__ void __launch_bounds__(256) k_q16x2_rank(const uint4* __restrict__ lines, const uint32_t* __restrict__ super,
                                                    const uint64_t* __restrict__ pack, uint32_t words, uint32_t half,
                                                    const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                                                    uint64_t* __restrict__ out, uint64_t m, uint64_t last_line,
                                                    unsigned long long* ctr) {
  extern __shared__ uint64_t lt_smem[];
  if (SRC == 1) lane_preload(pack, words, lt_smem);
  const uint32_t u = sc_unit_in_warp<32>();
  ScSched sc = sc_first<K, DYN, 32>(ctr);
  uint64_t qn[K];
  uint32_t cn[K];
  sc_load_qc<K, MODE == 0>(q, cs, sc.gb + u, sc.stride, m, qn, cn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, stride = sc.stride;
    uint64_t w[K][4];
    uint32_t xx[K], jj[K], cc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint32_t j, h, x;
      q16x2_locate(qn[k], last_line, j, h, x);
      xx[k] = x; jj[k] = j; cc[k] = MODE == 0 ? cn[k] : 0u;
      ld_sector_na(lines + 4 * (uint64_t)j + 2 * h, w[k][0], w[k][1], w[k][2], w[k][3]);
    }
    sc = sc_next<K, DYN, 32>(sc, ctr);
    sc_load_qc<K, MODE == 0>(q, cs, sc.gb + u, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      if (idx >= m) continue;
      const uint32_t sb = jj[k] >> QD_SB_LOG;
      if (MODE == 2) {
        st_stream_u64(out + idx, w[k][0] ^ w[k][1] ^ w[k][2] ^ w[k][3]);
      } else if (MODE == 0) {
        const uint32_t c = cc[k];
        const uint32_t s = SRC == 1 ? qd_s_field(qd_group_local(lt_smem, half, sb >> 3)[c], sb & 7u)
                                    : __ldg(super + 4 * sb + c);
        st_stream_u64(out + idx, q16x2_rank1(w[k], xx[k], c, s));
      } else {
        uint32_t s4[4];
        if (SRC == 1) {
          const uint64_t* grp = qd_group_local(lt_smem, half, sb >> 3);
#pragma unroll
          for (int c = 0; c < 4; ++c) s4[c] = qd_s_field(grp[c], sb & 7u);
        } else {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(super) + sb);
          s4[0] = v.x; s4[1] = v.y; s4[2] = v.z; s4[3] = v.w;
        }
        uint64_t r[4];
        q16x2_rank4(w[k], xx[k], s4, r);
        st_stream_v4u64(out + 4 * idx, r[0], r[1], r[2], r[3]);
      }
    }
  }
}

template <int K, int THREADS, int MODE, bool DYN>   // MODE 0 rank, 1 rank_4
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_q16x2_rank_c(const uint4* __restrict__ lines, const uint64_t* __restrict__ pack, uint64_t half_words,
                   const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs, uint64_t* __restrict__ out, uint64_t m,
                   uint64_t last_line, unsigned long long* ctr) {
  extern __shared__ uint64_t sc_smem[];
  uint32_t base0, base1;
  sc_preload(pack, half_words, sc_smem, base0, base1);
  const uint32_t u = sc_unit_in_warp<32>();
  ScSched sc = sc_first<K, DYN, 32>(ctr);
  uint64_t qn[K];
  uint32_t cn[K];
  sc_load_qc<K, MODE == 0>(q, cs, sc.gb + u, sc.stride, m, qn, cn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, stride = sc.stride;
    uint64_t w[K][4];
    uint32_t xx[K], cc[K], s[K][MODE == 0 ? 1 : 4];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      uint32_t j, h, x;
      q16x2_locate(qn[k], last_line, j, h, x);
      xx[k] = x; cc[k] = MODE == 0 ? cn[k] : 0u;
      ld_sector_na(lines + 4 * (uint64_t)j + 2 * h, w[k][0], w[k][1], w[k][2], w[k][3]);
      const uint32_t sb = j >> QD_SB_LOG, g = sb >> 3;
      const uint32_t addr = ((g & 1u) ? base1 : base0) + (g >> 1) * 32u;
      if (MODE == 0) {
        s[k][0] = qd_s_field(ld_dsmem_u64(addr + 8u * cc[k]), sb & 7u);
      } else {
        uint64_t v0, v1, v2, v3;
        ld_dsmem_v2u64(addr, v0, v1);
        ld_dsmem_v2u64(addr + 16u, v2, v3);
        s[k][MODE == 0 ? 0 : 0] = qd_s_field(v0, sb & 7u);
        s[k][MODE == 0 ? 0 : 1] = qd_s_field(v1, sb & 7u);
        s[k][MODE == 0 ? 0 : 2] = qd_s_field(v2, sb & 7u);
        s[k][MODE == 0 ? 0 : 3] = qd_s_field(v3, sb & 7u);
      }
    }
    sc = sc_next<K, DYN, 32>(sc, ctr);
    sc_load_qc<K, MODE == 0>(q, cs, sc.gb + u, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * stride;
      if (idx >= m) continue;
      if (MODE == 0) {
        st_stream_u64(out + idx, q16x2_rank1(w[k], xx[k], cc[k], s[k][0]));
      } else {
        uint32_t s4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) s4[c] = s[k][MODE == 0 ? 0 : c];
        uint64_t r[4];
        q16x2_rank4(w[k], xx[k], s4, r);
        st_stream_v4u64(out + 4 * idx, r[0], r[1], r[2], r[3]);
      }
    }
  }
  cluster_barrier();
}

// ------------------------------------------------------------------ launchers

extern int g_rank_k;
extern int g_index64;
extern int g_rank_smem;
extern int g_rank_pair;

// grid: as many 2-CTA clusters as fit at once (one CTA per SM); cached per (kernel, smem, device).
// The kernel's dynamic shared-memory limit only ever grows (a later, smaller table must not lower
// it below what a cached larger launch needs).
template <typename Kern>
static unsigned sc_grid(Kern kern, int threads, size_t smem, int device, int sms) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, size_t, int>, unsigned> cache;
  smem_limit_raise((const void*)kern, smem, device);
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple((const void*)kern, smem, device);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(sms & ~1));
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters <= 0) {
    cudaGetLastError();
    clusters = sms / 2;
  }
  return cache[key] = 2u * (unsigned)clusters;
}

// Co-resident 2-CTA clusters of the BiRank rank kernel at this handle's table size (diagnostics).
int super_pack_clusters(const qr_index* h) {
  if (!h->spack) return 0;
  auto kern = k_bi_rank2c<4, 1024, false, 2>;
  return (int)(sc_grid(kern, 1024, super_pack_cta_bytes(h), h->device, h->sm_count) / 2);
}

int l2_bytes(int device);

// Kernel shape of a rank / rank_4 launch (measured crossovers in
// profiles/r01_regime_probe.jsonl):
//   LANE    — one lane per query, superblock word from L2: best while the line array is mostly
//             L2-resident (<= 0.6 x L2: 135 vs 98 Gq/s for lane pairs at 33 MB);
//   PAIR    — lane pairs (one L2 request per line), global superblock words, dynamic order:
//             best up to ~2.2 x L2 (264 MB: 62 vs 54 Gq/s for the cluster kernel);
//   CLUSTER — lane pairs with the superblock words in 2-CTA cluster shared memory: best on
//             HBM-resident structures (2 GB: 46.2 vs 38.8 Gq/s), batches >= 2^22.
// Knobs: rank_pair 0 = always LANE, 1 = PAIR / CLUSTER by rank_smem only, 2 = by size (default);
// rank_smem 0 = never CLUSTER, 1 = by size and batch, 2 = whenever the table exists.
int rank_shape(const qr_index* h, uint64_t m) {
  if (g_rank_pair == 0) return RANK_LANE;
  const bool can = h->spack && !g_index64;
  if (can && g_rank_smem == 2) return RANK_CLUSTER;
  const double lines = (double)h->n_lines * 64.0, l2 = (double)l2_bytes(h->device);
  if (g_rank_pair == 2 && lines <= 0.6 * l2) return RANK_LANE;
  if (can && g_rank_smem == 1 && m >= (1ull << 22) && (g_rank_pair == 1 || lines > 2.2 * l2)) return RANK_CLUSTER;
  return RANK_PAIR;
}

extern int g_rank_dyn;
extern int g_rank_lane_table;
extern int g_rank_smem_k;
extern int g_rank_smem_threads;

extern int g_rank_smem_clusters;

template <typename Kern, typename... Args>
static void sc_go(Kern kern, int threads, const qr_index* h, size_t smem, cudaStream_t st, Args... args) {
  unsigned grid = sc_grid(kern, threads, smem, h->device, h->sm_count);
  if (g_rank_smem_clusters > 0) grid = 2u * (unsigned)g_rank_smem_clusters;
  kern<<<grid, threads, smem, st>>>(args...);
}

// (K, threads per CTA): in-flight queries per SM = threads / 2 * K; registers per thread are
// capped at 65536 / threads by the one-CTA-per-SM launch bound.
template <int K, int T>
static void sc_launch_kt(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m, int what,
                         unsigned long long* ctr, bool dyn, cudaStream_t st) {
  const size_t smem = super_pack_cta_bytes(h);
  const uint64_t hw = h->spack_half * (h->sigma == 2 ? 1 : 4);     // u64 words per CTA
  const uint64_t last = h->n_lines - 1;
  const uint4* L = h->lines;
  const uint64_t* P = h->spack;
  if (h->sigma == 2) {
    if (c) {
      if (dyn) sc_go(k_bi_rank2c<K, T, true, 2>, T, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
      else     sc_go(k_bi_rank2c<K, T, true, 0>, T, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
    } else if (what == 3) {
      if (dyn) sc_go(k_bi_rank2c<K, T, false, 3>, T, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
      else     sc_go(k_bi_rank2c<K, T, false, 1>, T, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
    } else {
      if (dyn) sc_go(k_bi_rank2c<K, T, false, 2>, T, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
      else     sc_go(k_bi_rank2c<K, T, false, 0>, T, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
    }
  } else if (what == 0) {
    if (dyn) sc_go(k_qd_rank2c<K, T, true>, T, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
    else     sc_go(k_qd_rank2c<K, T, false>, T, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
  } else {
    if (dyn) sc_go(k_qd_all4_2c<K, T, true>, T, h, smem, st, L, P, hw, q, out, m, last, ctr);
    else     sc_go(k_qd_all4_2c<K, T, false>, T, h, smem, st, L, P, hw, q, out, m, last, ctr);
  }
}

// One-lane kernels with the per-CTA table (rank_shape LANE).  Returns cudaErrorNotSupported when
// the handle has no table small enough (the caller then uses the global-memory lane kernels).
extern int g_rank_resident;

// largest dynamic shared memory per CTA this device allows (opt-in), capped at 200 KB
static uint64_t res_max_bytes(int device) {
  static std::mutex mu;
  static std::map<int, uint64_t> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess || v <= 0) {
    cudaGetLastError();
    v = 0;
  }
  const uint64_t r = (uint64_t)v < 200 * 1024 ? (uint64_t)v : 200 * 1024;
  return cache[device] = r;
}


cudaError_t launch_lane_table_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                   int what, cudaStream_t st) {
  if (!h->spack || g_index64) return cudaErrorNotSupported;
  const uint64_t total = 2 * super_pack_cta_bytes(h);
  if (total > LANE_TABLE_MAX) return cudaErrorNotSupported;
  const uint32_t words = (uint32_t)(total / 8), half = (uint32_t)h->spack_half;
  const uint64_t last = h->n_lines - 1;
  const bool dyn = use_dyn_order(m);
  constexpr int K = 2;
  // resident structure: table + lines in every CTA's shared memory, when it fits and the batch
  // moves at least 2x the bytes the preload reads (one copy per SM; 16 B of query I/O per query).
  // Measured crossover (profiles/r01_small_probe.jsonl): at 135 KB, 10^6 queries lose (59 vs 68
  // Gq/s from L2) and 10^7 win (128 vs 93); at 17 KB 10^6 already win (68 vs 36: the L2 path
  // hot-spots on the few lines every query hits)
  const uint64_t res_bytes = total + h->n_lines * 64;
  if (g_rank_resident && (total % 16) == 0 && res_bytes <= res_max_bytes(h->device) &&
      m * 16 >= 2 * res_bytes * (uint64_t)h->sm_count) {
    const unsigned grid = (unsigned)h->sm_count;                 // one 1024-thread CTA per SM
    auto go_res = [&](auto kern, const uint8_t* cc) -> cudaError_t {
      smem_limit_raise((const void*)kern, (size_t)res_bytes, h->device);
      kern<<<grid, 1024, (size_t)res_bytes, st>>>(h->lines, h->spack, words, half, q, cc, out, m, last, nullptr);
      return cudaGetLastError();
    };
    if (h->sigma == 2) return c ? go_res(k_bi_rank1s<K, true, false, true>, c) : go_res(k_bi_rank1s<K, false, false, true>, c);
    if (what == 0) return go_res(k_qd_rank1s<K, 0, false, true>, c);
    return go_res(k_qd_rank1s<K, 1, false, true>, nullptr);
  }
  const unsigned g = grid_stride_blocks((m + K - 1) / K, 256, h->sm_count, g_rank_blocks_per_sm);
  const uint4* L = h->lines;
  const uint64_t* P = h->spack;
  auto go = [&](auto ks, auto kd, const uint8_t* cc) -> cudaError_t {
    return launch_ordered_smem(ks, kd, dyn, h->device, h->sm_count, g, (size_t)total, st, L, P, words, half, q, cc, out,
                               m, last);
  };
  if (h->sigma == 2) {
    if (c) return go(k_bi_rank1s<K, true, false>, k_bi_rank1s<K, true, true>, c);
    return go(k_bi_rank1s<K, false, false>, k_bi_rank1s<K, false, true>, c);
  }
  if (what == 0) return go(k_qd_rank1s<K, 0, false>, k_qd_rank1s<K, 0, true>, c);
  return go(k_qd_rank1s<K, 1, false>, k_qd_rank1s<K, 1, true>, nullptr);
}

// Launch a 1024-thread kernel over CS-CTA clusters (cluster size at launch time; 16 needs the
// non-portable opt-in), as many clusters as the occupancy API allows at `smem` bytes per CTA
// (cached per kernel, device, CS and size), with a leased work counter as the last argument.
template <typename... KArgs, typename... Args>
static cudaError_t launch_cs_clusters(void (*kern)(KArgs...), uint32_t cs, size_t smem, const qr_index* h,
                                      cudaStream_t st, Args... args) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, uint32_t, size_t>, unsigned> grids;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cs; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  unsigned grid = 0;
  // the limit is raised before EVERY launch (a smaller table of another handle may have been
  // launched since this key was cached); it only ever grows, so concurrent launches stay valid
  smem_limit_raise((const void*)kern, smem, h->device);
  {
    std::lock_guard<std::mutex> g(mu);
    const auto key = std::make_tuple((const void*)kern, h->device, cs, smem);
    auto it = grids.find(key);
    if (it != grids.end()) {
      grid = it->second;
    } else {
      if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cfg.gridDim = dim3((unsigned)h->sm_count / cs * cs);
      int clusters = 0;
      if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters <= 0) {
        cudaGetLastError();
        clusters = 1;
      }
      grid = grids[key] = (unsigned)clusters * cs;
    }
  }
  CounterLease lease;
  unsigned long long* ctr = nullptr;
  cudaError_t e = lease.acquire(h->device, st, &ctr);
  if (e) return e;
  cfg.gridDim = dim3(grid);
  cfg.stream = st;
  e = cudaLaunchKernelEx(&cfg, kern, args..., ctr);
  if (!e) e = cudaGetLastError();
  cudaError_t e2 = lease.release(st);
  return e ? e : e2;
}

static uint32_t cs_log_of(uint32_t cs) { return cs == 4 ? 2 : cs == 8 ? 3 : 4; }

// BiRank16 rank over the CS-CTA table (h->spack_big): dynamic order, one 1024-thread CTA per SM.
cudaError_t launch_big_pack_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                 cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const uint32_t cs = h->spack_big_cs;
  const size_t smem = (size_t)h->spack_big_slots * 8;
  const uint4* L = h->lines;
  const uint64_t* P = h->spack_big;
  const uint64_t slots = h->spack_big_slots, last = h->n_lines - 1;
  const uint32_t* hb = h->spack_big_hi;
  if (c)
    return launch_cs_clusters(k_bi_rank2v<4, 1024, true>, cs, smem, h, st, L, P, slots, cs_log_of(cs), hb[0], hb[1], hb[2],
                              q, c, out, m, last);
  return launch_cs_clusters(k_bi_rank2v<4, 1024, false>, cs, smem, h, st, L, P, slots, cs_log_of(cs), hb[0], hb[1], hb[2],
                            q, c, out, m, last);
}

// QuadRank16 rank (what 0) / rank_4 (what 1) over the CS-CTA table
cudaError_t launch_big_pack_qd(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                               int what, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const uint32_t cs = h->spack_big_cs;
  const uint64_t part_words = h->spack_big_slots * 4, last = h->n_lines - 1;
  const size_t smem = (size_t)part_words * 8;
  const uint4* L = h->lines;
  const uint64_t* P = h->spack_big;
  if (what) return launch_cs_clusters(k_qd_all4_2w<2, 1024>, cs, smem, h, st, L, P, part_words, cs_log_of(cs), q, out, m, last);
  return launch_cs_clusters(k_qd_rank2w<2, 1024>, cs, smem, h, st, L, P, part_words, cs_log_of(cs), q, c, out, m, last);
}

// what: 0 = rank (sigma 2 or 4), 1 = rank_4 (sigma 4), 3 = BiRank gather ceiling of this kernel shape
cudaError_t launch_super_pack_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                   int what, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const bool dyn = g_rank_dyn != 0;
  CounterLease lease;
  unsigned long long* ctr = nullptr;
  cudaError_t e;
  if (dyn && (e = lease.acquire(h->device, st, &ctr))) return e;
  // default K (measured, profiles/r01_smem_probe_k.jsonl): BiRank 4 (fits 64 registers), QuadRank 2
  // (K = 4 spills at the 64-register cap of 1024-thread CTAs)
  const int k = g_rank_smem_k ? g_rank_smem_k : (h->sigma == 2 ? 4 : 2);
  const int t = g_rank_smem_threads ? g_rank_smem_threads : (k == 6 ? 768 : k == 8 ? 512 : 1024);
  switch (k * 10000 + t) {
    case 11024: sc_launch_kt<1, 1024>(h, q, c, out, m, what, ctr, dyn, st); break;
    case 21024: sc_launch_kt<2, 1024>(h, q, c, out, m, what, ctr, dyn, st); break;
    case 31024: sc_launch_kt<3, 1024>(h, q, c, out, m, what, ctr, dyn, st); break;
    case 40768: sc_launch_kt<4, 768>(h, q, c, out, m, what, ctr, dyn, st); break;
    case 60768: sc_launch_kt<6, 768>(h, q, c, out, m, what, ctr, dyn, st); break;
    case 80512: sc_launch_kt<8, 512>(h, q, c, out, m, what, ctr, dyn, st); break;
    case 41024: sc_launch_kt<4, 1024>(h, q, c, out, m, what, ctr, dyn, st); break;
    default: break;   // not instantiated: rejected by qr_set_tuning's pair check
  }
  e = cudaGetLastError();
  if (dyn) {
    cudaError_t e2 = lease.release(st);
    if (!e) e = e2;
  }
  return e;
}


// BiRank16x2 dispatch (what: 0 rank, 2 gather ceiling).  Superblock-word source by structure
// size, as rank_shape: per-CTA table while the line array is L2-resident and the table small;
// cluster shared memory for HBM-resident arrays and batches >= 2^22 (rank_smem); else L2.
cudaError_t launch_b16x2_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                              int what, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  constexpr int K = 4;
  const uint64_t last = h->n_lines - 1;
  const bool dyn = use_dyn_order(m);
  const unsigned g = grid_stride_blocks((m + K - 1) / K, 256, h->sm_count, g_rank_blocks_per_sm);
  const uint4* L = h->lines;
  const uint32_t* S = h->super;
  const uint64_t table = h->spack ? 2 * super_pack_cta_bytes(h) : 0;
  const double lines = (double)h->n_lines * 64.0, l2 = (double)l2_bytes(h->device);
  if (what == 2)
    return launch_ordered(k_b16x2_rank<K, 0, 1, false, false>, k_b16x2_rank<K, 0, 1, false, true>, dyn, h->device,
                          h->sm_count, g, st, L, S, h->spack, 0u, 0u, q, c, out, m, last);
  const bool can_cluster = h->spack && !g_index64;
  const bool cluster = can_cluster && (g_rank_smem == 2 || (g_rank_smem == 1 && m >= (1ull << 22) && lines > 0.6 * l2));
  if (cluster) {
    CounterLease lease;
    unsigned long long* ctr = nullptr;
    cudaError_t e;
    if (g_rank_dyn && (e = lease.acquire(h->device, st, &ctr))) return e;
    const size_t smem = super_pack_cta_bytes(h);
    const uint64_t hw = h->spack_half;
    if (c) {
      if (ctr) sc_go(k_b16x2_rank_c<K, 1024, true, true>, 1024, h, smem, st, L, h->spack, hw, q, c, out, m, last, ctr);
      else     sc_go(k_b16x2_rank_c<K, 1024, true, false>, 1024, h, smem, st, L, h->spack, hw, q, c, out, m, last, ctr);
    } else {
      if (ctr) sc_go(k_b16x2_rank_c<K, 1024, false, true>, 1024, h, smem, st, L, h->spack, hw, q, c, out, m, last, ctr);
      else     sc_go(k_b16x2_rank_c<K, 1024, false, false>, 1024, h, smem, st, L, h->spack, hw, q, c, out, m, last, ctr);
    }
    e = cudaGetLastError();
    if (ctr) {
      cudaError_t e2 = lease.release(st);
      if (!e) e = e2;
    }
    return e;
  }
  if (h->spack && table <= LANE_TABLE_MAX && g_rank_lane_table) {
    const uint32_t words = (uint32_t)(table / 8), half = (uint32_t)h->spack_half;
    if (c) return launch_ordered_smem(k_b16x2_rank<K, 1, 0, true, false>, k_b16x2_rank<K, 1, 0, true, true>, dyn, h->device,
                                      h->sm_count, g, (size_t)table, st, L, S, h->spack, words, half, q, c, out, m, last);
    return launch_ordered_smem(k_b16x2_rank<K, 1, 0, false, false>, k_b16x2_rank<K, 1, 0, false, true>, dyn, h->device,
                               h->sm_count, g, (size_t)table, st, L, S, h->spack, words, half, q, c, out, m, last);
  }
  if (c) return launch_ordered(k_b16x2_rank<K, 0, 0, true, false>, k_b16x2_rank<K, 0, 0, true, true>, dyn, h->device,
                               h->sm_count, g, st, L, S, h->spack, 0u, 0u, q, c, out, m, last);
  return launch_ordered(k_b16x2_rank<K, 0, 0, false, false>, k_b16x2_rank<K, 0, 0, false, true>, dyn, h->device,
                        h->sm_count, g, st, L, S, h->spack, 0u, 0u, q, c, out, m, last);
}


// QuadRank16x2 dispatch (what: 0 rank, 1 rank_4, 2 gather ceiling); superblock source as BiRank16x2.
cudaError_t launch_q16x2_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                              int what, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  constexpr int K = 2;
  const uint64_t last = h->n_lines - 1;
  const bool dyn = use_dyn_order(m);
  const unsigned g = grid_stride_blocks((m + K - 1) / K, 256, h->sm_count, g_rank_blocks_per_sm);
  const uint4* L = h->lines;
  const uint32_t* S = h->super;
  const uint64_t table = h->spack ? 2 * super_pack_cta_bytes(h) : 0;
  const double lines = (double)h->n_lines * 64.0, l2 = (double)l2_bytes(h->device);
  if (what == 2)
    return launch_ordered(k_q16x2_rank<K, 0, 2, false>, k_q16x2_rank<K, 0, 2, true>, dyn, h->device, h->sm_count, g, st,
                          L, S, h->spack, 0u, 0u, q, c, out, m, last);
  const bool can_cluster = h->spack && !g_index64;
  const bool cluster = can_cluster && (g_rank_smem == 2 || (g_rank_smem == 1 && m >= (1ull << 22) && lines > 0.6 * l2));
  if (cluster) {
    CounterLease lease;
    unsigned long long* ctr = nullptr;
    cudaError_t e;
    if (g_rank_dyn && (e = lease.acquire(h->device, st, &ctr))) return e;
    const size_t smem = super_pack_cta_bytes(h);
    const uint64_t hw = 4 * h->spack_half;
    const uint64_t* P = h->spack;
    if (what == 0) {
      if (ctr) sc_go(k_q16x2_rank_c<K, 1024, 0, true>, 1024, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
      else     sc_go(k_q16x2_rank_c<K, 1024, 0, false>, 1024, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
    } else {
      if (ctr) sc_go(k_q16x2_rank_c<K, 1024, 1, true>, 1024, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
      else     sc_go(k_q16x2_rank_c<K, 1024, 1, false>, 1024, h, smem, st, L, P, hw, q, c, out, m, last, ctr);
    }
    e = cudaGetLastError();
    if (ctr) {
      cudaError_t e2 = lease.release(st);
      if (!e) e = e2;
    }
    return e;
  }
  if (h->spack && table <= LANE_TABLE_MAX && g_rank_lane_table) {
    const uint32_t words = (uint32_t)(table / 8), half = (uint32_t)h->spack_half;
    if (what == 0)
      return launch_ordered_smem(k_q16x2_rank<K, 1, 0, false>, k_q16x2_rank<K, 1, 0, true>, dyn, h->device, h->sm_count, g,
                                 (size_t)table, st, L, S, h->spack, words, half, q, c, out, m, last);
    return launch_ordered_smem(k_q16x2_rank<K, 1, 1, false>, k_q16x2_rank<K, 1, 1, true>, dyn, h->device, h->sm_count, g,
                               (size_t)table, st, L, S, h->spack, words, half, q, c, out, m, last);
  }
  if (what == 0)
    return launch_ordered(k_q16x2_rank<K, 0, 0, false>, k_q16x2_rank<K, 0, 0, true>, dyn, h->device, h->sm_count, g, st,
                          L, S, h->spack, 0u, 0u, q, c, out, m, last);
  return launch_ordered(k_q16x2_rank<K, 0, 1, false>, k_q16x2_rank<K, 0, 1, true>, dyn, h->device, h->sm_count, g, st,
                        L, S, h->spack, 0u, 0u, q, c, out, m, last);
}


// BiRank32x2 dispatch (what: 0 rank, 2 gather ceiling).
cudaError_t launch_b32x2_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                              int what, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  constexpr int K = 4;
  const uint64_t last = h->n_lines - 1;
  const bool dyn = use_dyn_order(m);
  const unsigned g = grid_stride_blocks((m + K - 1) / K, 256, h->sm_count, g_rank_blocks_per_sm);
  const uint4* L = h->lines;
  const uint64_t* l1 = reinterpret_cast<const uint64_t*>(h->super);
  const uint32_t words = (uint32_t)h->n_super;
  const size_t smem = ((size_t)words * 8 + 15) & ~(size_t)15;
  if (what == 2)
    return launch_ordered_smem(k_b32x2_rank<K, 1, false, false>, k_b32x2_rank<K, 1, false, true>, dyn, h->device,
                               h->sm_count, g, smem, st, L, l1, words, q, c, out, m, last);
  if (c)
    return launch_ordered_smem(k_b32x2_rank<K, 0, true, false>, k_b32x2_rank<K, 0, true, true>, dyn, h->device,
                               h->sm_count, g, smem, st, L, l1, words, q, c, out, m, last);
  return launch_ordered_smem(k_b32x2_rank<K, 0, false, false>, k_b32x2_rank<K, 0, false, true>, dyn, h->device,
                             h->sm_count, g, smem, st, L, l1, words, q, c, out, m, last);
}

}  // namespace qr
