// fm.cu — QuadFm (App. D) on sm_100a.
//
// Build: suffix array of T$ on the GPU by prefix doubling over device radix sorts (the
// paper leaves SA construction implicit), the BWT with '$' stored as A
// and its row spos kept, C[c] = 1 + #{t_i < c}, QuadRank16 over the
// N = n+1 BWT symbols (quadrank.cu), and the 8-mer interval table.
//
// Count: backward search: [lo,hi) from the 8-mer table (or [0,N)), then
// for each remaining pattern char c right to left: lo = C[c] + Occ(c,lo), hi = C[c] + Occ(c,hi)
// with Occ(c,x) = rank(x,c) - [c = A and x > spos]; stop when lo >= hi.  One pattern per lane;
// a lane refills itself from its grid-stride pattern sequence as soon as its pattern finishes,
// so lanes never wait for the slowest pattern of a static batch (the GPU analogue of the
// paper's swap-pop active list).
#include <algorithm>
#include <mutex>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <type_traits>

#include "qr_common.cuh"

namespace qr {

struct FmParams {
  const uint4* lines;
  const uint32_t* super;
  const uint2* kmer;
  int K;                // k-mer table width (0: no table)
  uint64_t spos;
  uint64_t N;
  uint64_t last_line;
  uint32_t C[4];        // host copy; the kernels read C from the table tail (Ct) with one load
  const uint32_t* Ct;   // = (const uint32_t*)(kmer + 4^K): C[0..3] stored after the k-mer table
  int bw;                 // BWT rank layout: 0 QuadRank16, 1 QuadRank16x2 (sector-local)
  const uint64_t* spack;  // packed superblock table (sbcache.cu encoding, 2 parts), or null
  uint32_t spack_half;    // groups per part
  uint32_t n_super;
  const uint32_t* kbits;  // approximate search: presence bitmap of the table (4^K bits), or null
};

// Superblock word s_{sb,c}.  SMS 0: global memory (an L2 request per read);
// SMS 1: the raw u32 x 4 array copied into shared memory at CTA start; SMS 2: the packed table
// (sbcache.cu: 8 superblocks per u64 per symbol) copied into shared memory.  The FM step reads
// s twice (lo and hi), so 1 and 2 remove up to two L2 requests / L1 wavefront sets per step.
template <int SMS>
__device__ __forceinline__ uint32_t fm_super(const FmParams& F, uint32_t sb, uint32_t c) {
  if (SMS == 0) return __ldg(F.super + 4 * sb + c);
  extern __shared__ uint64_t fm_smem[];
  if (SMS == 1) return reinterpret_cast<const uint32_t*>(fm_smem)[4 * sb + c];
  const uint32_t g = sb >> 3, k = sb & 7u;
  const uint64_t v = fm_smem[4 * ((g & 1u) * F.spack_half + (g >> 1)) + c];
  const uint32_t lo = (uint32_t)v & 0x3fffffu;
  return k ? lo + ((uint32_t)(v >> (16u + 6u * k)) & 0x3fu) : lo;
}

template <int SMS>
__device__ __forceinline__ void fm_preload_super(const FmParams& F) {
  if (SMS == 0) return;
  extern __shared__ uint64_t fm_smem[];
  const uint4* src = reinterpret_cast<const uint4*>(SMS == 1 ? reinterpret_cast<const uint64_t*>(F.super) : F.spack);
  const uint32_t n16 = SMS == 1 ? F.n_super : 4u * F.spack_half;       // 16-B units
  uint4* dst = reinterpret_cast<uint4*>(fm_smem);
  for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldg(src + i);
  __syncthreads();
}

__device__ __forceinline__ uint32_t text_char(const uint64_t* t, uint64_t i) {
  return (uint32_t)(t[i >> 5] >> (2 * (i & 31))) & 3u;
}

// ------------------------------------------------------------------ SA by prefix doubling

// initial key: the first 21 characters, 3 bits each ($ and beyond = 0, A..T = 1..4), MSB first
__global__ void k_sa_init(const uint64_t* __restrict__ text, uint64_t n, uint64_t* __restrict__ keys,
                          uint32_t* __restrict__ vals) {
  const uint64_t N = n + 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t key = 0;
#pragma unroll
    for (int t = 0; t < 21; ++t) {
      uint64_t x = i + t;
      uint64_t code = x < n ? (uint64_t)text_char(text, x) + 1 : 0;
      key = (key << 3) | code;
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
  }
}

// Prefix doubling with discarding.  Every round sorts only the ACTIVE suffixes — those whose
// group (equal first h characters) still has more than one member — by (group start, rank of the
// suffix h further on); suffixes in singleton groups are final and never touched again.  rank[i]
// is the sorted position of the first member of suffix i's group (its group start), so for a
// singleton it is its final SA position; pos[k] is the SA position the k-th active item occupies
// (increasing in k, and each group is a contiguous run), so after a round's sort the k-th item
// lands at SA[pos[k]].  On the block-repeat text of configs[4] ~39% of the suffixes survive the
// first round and ~1% the fifth, against a full 2^30-item sort in every round before.

// pos == nullptr: the identity (round 0, every suffix active in SA order)
__device__ __forceinline__ uint32_t sa_pos(const uint32_t* __restrict__ pos, uint64_t k) {
  return pos ? pos[k] : (uint32_t)k;
}

__device__ __forceinline__ bool sa_head(const uint64_t* __restrict__ K, uint64_t k) {
  return k == 0 || K[k] != K[k - 1];
}

// gs[k] = pos[k] if sorted active item k starts a new group, else 0 (max-scanned into group starts)
__global__ void k_sa_heads(const uint64_t* __restrict__ K, const uint32_t* __restrict__ pos, uint64_t A,
                           uint32_t* __restrict__ gs) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < A; k += (uint64_t)gridDim.x * blockDim.x)
    gs[k] = sa_head(K, k) ? sa_pos(pos, k) : 0u;
}

struct MaxU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

// Place the sorted active items: SA[pos[k]] = V[k], rank[V[k]] = its new group start (rounds
// after the first write it only where it changed: the group's first subgroup keeps the old start,
// the key's high part); flag[k] = 1 while item k's group still has another member (stays active).
__global__ void k_sa_place(const uint64_t* __restrict__ K, const uint32_t* __restrict__ V,
                           const uint32_t* __restrict__ pos, const uint32_t* __restrict__ gs, uint64_t A,
                           int gshift, uint32_t* __restrict__ sa, uint32_t* __restrict__ rank,
                           uint32_t* __restrict__ flag) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < A; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = V[k], g = gs[k];
    const uint64_t key = K[k];
    sa[sa_pos(pos, k)] = v;
    if (gshift == 0 || (uint32_t)(key >> gshift) != g) rank[v] = g;
    const bool single = (k == 0 || key != K[k - 1]) && (k + 1 == A || K[k + 1] != key);
    flag[k] = single ? 0u : 1u;
  }
}

// Keep the active items, in SA-position order: survivor k goes to slot off[k] (off = the
// exclusive sum of flag) with its SA position, group start and suffix index, so the next
// round's keys read them sequentially; the count of survivors goes to *count.
__global__ void k_sa_compact(const uint64_t* __restrict__ K, const uint32_t* __restrict__ V,
                             const uint32_t* __restrict__ pos, const uint32_t* __restrict__ gs,
                             const uint32_t* __restrict__ off, uint64_t A, uint32_t* __restrict__ pos_out,
                             uint32_t* __restrict__ g_out, uint32_t* __restrict__ i_out,
                             unsigned long long* __restrict__ count) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < A; k += (uint64_t)gridDim.x * blockDim.x) {
    const bool single = sa_head(K, k) && (k + 1 == A || K[k + 1] != K[k]);
    if (!single) {
      const uint32_t o = off[k];
      pos_out[o] = sa_pos(pos, k);
      g_out[o] = gs[k];
      i_out[o] = V[k];
    }
    if (k + 1 == A) *count = (unsigned long long)off[k] + (single ? 0u : 1u);
  }
}

// survivors of a round from the exclusive sum of its flags: off[A-1] + [item A-1 stays active]
__global__ void k_sa_survivors(const uint64_t* __restrict__ K, const uint32_t* __restrict__ off, uint64_t A,
                               unsigned long long* __restrict__ count) {
  const uint64_t k = A - 1;
  const bool single = sa_head(K, k) && (k + 1 == A || K[k + 1] != K[k]);
  *count = (unsigned long long)off[k] + (single ? 0u : 1u);
}

// doubling key of active item k (suffix i = ii[k], group start gg[k]): (gg[k], rank of the suffix
// h further on + 1, or 0 past the end), packed in 2*b bits
__global__ void k_sa_keys(const uint32_t* __restrict__ gg, const uint32_t* __restrict__ ii,
                          const uint32_t* __restrict__ rank, uint64_t A, uint64_t N, uint64_t h, int b,
                          uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < A; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = ii[k];
    const uint64_t r2 = ((uint64_t)i + h < N) ? (uint64_t)rank[i + h] + 1 : 0;
    keys[k] = ((uint64_t)gg[k] << b) | r2;
    vals[k] = i;
  }
}

static int bits_for(uint64_t x) {  // bits needed to represent values 0..x
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b ? b : 1;
}

// d_sa: N u32 outputs.  The temporaries (32 B per suffix + the sort's scratch, then 8 B per
// survivor of round 0) are
// cudaMalloc arenas: the stream-ordered pool maps and unmaps large blocks ~50x slower (43 GB:
// 0.27 s to map and 0.26-1.2 s to release vs 0.004 / 0.01 s, profiles/r01_alloc_probe.jsonl).
// The caller's stream is synchronised every round (survivor count) and before the free.
static qr_status build_sa(const uint64_t* d_text, uint64_t n, int sms, cudaStream_t st, uint32_t* d_sa) {
  const uint64_t N = n + 1;
  uint64_t *ka = nullptr, *kb = nullptr;
  uint32_t *va = nullptr, *vb = nullptr, *rank = nullptr, *gs = nullptr, *pa = nullptr, *pb = nullptr;
  unsigned long long* count = nullptr;
  unsigned long long* h_count = nullptr;
  void* tmp = nullptr;
  char* arena = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  char* pos_arena = nullptr;             // the two survivor lists, sized after round 0
  auto cleanup = [&]() {
    if (arena || pos_arena) cudaStreamSynchronize(st);
    if (arena) cudaFree(arena);
    if (pos_arena) cudaFree(pos_arena);
    if (h_count) cudaFreeHost(h_count);
  };
  auto bail = [&](cudaError_t err, const char* what) { cleanup(); return cuda_fail(err, what); };
  {
    size_t need = 0, need2 = 0, need3 = 0;
    cub::DoubleBuffer<uint64_t> K(ka, kb);
    cub::DoubleBuffer<uint32_t> V(va, vb);
    if ((e = cub::DeviceRadixSort::SortPairs(nullptr, need, K, V, (int64_t)N, 0, 64, st))) return bail(e, "sort size");
    if ((e = cub::DeviceScan::InclusiveScan(nullptr, need2, gs, gs, MaxU32(), (int64_t)N, st))) return bail(e, "scan size");
    if ((e = cub::DeviceScan::ExclusiveSum(nullptr, need3, va, va, (int64_t)N, st))) return bail(e, "scan size");
    tmp_bytes = need > need2 ? need : need2;
    tmp_bytes = tmp_bytes > need3 ? tmp_bytes : need3;
  }
  const size_t u32N = (N * 4 + 255) & ~(size_t)255, u64N = (N * 8 + 255) & ~(size_t)255;
  const size_t arena_bytes = 2 * u64N + 4 * u32N + 256 + ((tmp_bytes + 255) & ~(size_t)255);
  if ((e = cudaMalloc((void**)&arena, arena_bytes))) { arena = nullptr; return bail(e, "sa scratch"); }
  if ((e = cudaMallocHost((void**)&h_count, 8))) return bail(e, "sa host count");
  {
    char* p = arena;
    ka = reinterpret_cast<uint64_t*>(p); p += u64N;
    kb = reinterpret_cast<uint64_t*>(p); p += u64N;
    uint32_t** u32s[4] = {&va, &vb, &rank, &gs};
    for (auto q : u32s) { *q = reinterpret_cast<uint32_t*>(p); p += u32N; }
    count = reinterpret_cast<unsigned long long*>(p); p += 256;
    tmp = p;
  }
  const int b = bits_for(N);
  auto grid = [&](uint64_t items) { return grid_stride_blocks(items, 256, sms, 16); };
  // round 0: every suffix active, keyed by its first 21 characters
  k_sa_init<<<grid(N), 256, 0, st>>>(d_text, n, ka, va);
  uint64_t A = N, h = 21;
  int bits = 63;
  uint64_t* kin = ka;                        // keys of the round are written here
  uint32_t* carry = nullptr;                 // survivors' group starts [0, N) and suffixes [N, 2N)
  for (int round = 0; round < 64 && A; ++round) {
    if (round) k_sa_keys<<<grid(A), 256, 0, st>>>(carry, carry + N, rank, A, N, h >> 1, b, kin, va);
    cub::DoubleBuffer<uint64_t> K(kin, kin == ka ? kb : ka);
    cub::DoubleBuffer<uint32_t> V(va, vb);
    size_t tb = tmp_bytes;
    if ((e = cub::DeviceRadixSort::SortPairs(tmp, tb, K, V, (int64_t)A, 0, bits, st))) return bail(e, "sort");
    k_sa_heads<<<grid(A), 256, 0, st>>>(K.Current(), round ? pa : nullptr, A, gs);
    tb = tmp_bytes;
    if ((e = cub::DeviceScan::InclusiveScan(tmp, tb, gs, gs, MaxU32(), (int64_t)A, st))) return bail(e, "scan");
    uint32_t* flag = V.Alternate();          // free after the sort; becomes the offsets
    k_sa_place<<<grid(A), 256, 0, st>>>(K.Current(), V.Current(), round ? pa : nullptr, gs, A, round ? b : 0, d_sa, rank,
                                        flag);
    tb = tmp_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, flag, flag, (int64_t)A, st))) return bail(e, "scan");
    carry = reinterpret_cast<uint32_t*>(K.Alternate());   // free after the sort: 2N u32
    if (round == 0) {
      // the survivor lists are sized by round 0's survivors (peak 32 + 8 * A1/N bytes per suffix
      // instead of 40, so that n up to 2^32 - 2 builds within a B200's HBM)
      k_sa_survivors<<<1, 1, 0, st>>>(K.Current(), flag, A, count);
      cudaMemcpyAsync(h_count, count, 8, cudaMemcpyDeviceToHost, st);
      if ((e = cudaStreamSynchronize(st))) return bail(e, "sa round sync");
      const size_t u32A = ((*h_count ? *h_count : 1) * 4 + 255) & ~(size_t)255;
      if ((e = cudaMalloc((void**)&pos_arena, 2 * u32A))) { pos_arena = nullptr; return bail(e, "sa positions"); }
      pb = reinterpret_cast<uint32_t*>(pos_arena);
      pa = reinterpret_cast<uint32_t*>(pos_arena + u32A);
    }
    k_sa_compact<<<grid(A), 256, 0, st>>>(K.Current(), V.Current(), round ? pa : nullptr, gs, flag, A, pb, carry,
                                          carry + N, count);
    cudaMemcpyAsync(h_count, count, 8, cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st))) return bail(e, "sa round sync");
    A = *h_count;
    uint32_t* t = pa; pa = pb; pb = t;
    kin = K.Current();                       // the next round's keys go to the buffer not holding `carry`
    h *= 2;                                  // keys of the next round look h/2 = this round's reach ahead
    bits = 2 * b;
  }
  if (A) return bail(cudaErrorUnknown, "sa: suffix sort did not converge");
  if ((e = cudaGetLastError())) return bail(e, "sa kernels");
  cleanup();
  return QR_OK;
}

// ------------------------------------------------------------------ BWT

// one output word (32 BWT symbols) per thread; '$' stored as A (0); spos recorded
__global__ void k_bwt(const uint64_t* __restrict__ text, const uint32_t* __restrict__ sa, uint64_t N,
                      uint64_t* __restrict__ bwt, unsigned long long* __restrict__ spos) {
  const uint64_t nw = (N + 31) >> 5;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = 0;
    for (uint64_t k = 0; k < 32 && 32 * w + k < N; ++k) {
      uint64_t s = sa[32 * w + k];
      if (s == 0) *spos = 32 * w + k;
      else x |= (uint64_t)text_char(text, s - 1) << (2 * k);
    }
    bwt[w] = x;
  }
}

// symbol counts of the text (first n chars): cnt[c]
__global__ void k_sym_counts(const uint64_t* __restrict__ text, uint64_t n, unsigned long long* __restrict__ cnt) {
  uint32_t a[4] = {0, 0, 0, 0};
  const uint64_t nw = (n + 31) >> 5;
  const uint64_t M = 0x5555555555555555ull;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = text[w];
    uint64_t valid = (32 * w + 32 <= n) ? 32 : n - 32 * w;
    uint64_t vm = valid == 32 ? M : (((1ull << (2 * valid)) - 1) & M);
    uint64_t lo = x & vm, hi = (x >> 1) & vm;
    uint32_t c3 = __popcll(lo & hi), l1 = __popcll(lo), h1 = __popcll(hi);
    a[3] += c3; a[1] += l1 - c3; a[2] += h1 - c3; a[0] += (uint32_t)valid - l1 - h1 + c3;
  }
  for (int c = 0; c < 4; ++c) {
    uint32_t v = a[c];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(cnt + c, (unsigned long long)v);
  }
}

// ------------------------------------------------------------------ rank inside the FM loop

// Prefix masks of every in-half position x (0..127) of a QuadRank16 BWT line, as a per-CTA
// shared table, for rank_4 and the steps of the issue-bound approximate search (+7.5% at k = 1)
// and the k-mer table build; the count kernels keep computing them (the table's shared loads
// cost the L1-bound configs[3] kernel wavefronts and the HBM kernels latency: -5% measured).
__shared__ __align__(16) uint64_t g_qd_masks[128][2];
__device__ __forceinline__ void qd_masks_init() {
  for (uint32_t i = threadIdx.x; i < 128; i += blockDim.x) {
    g_qd_masks[i][0] = prefix_mask((int)i, 0);
    g_qd_masks[i][1] = prefix_mask((int)i, 1);
  }
  __syncthreads();
}
__device__ __forceinline__ void qd_masks(uint32_t x, uint64_t& m0, uint64_t& m1) {
  const uint4 mm = reinterpret_cast<const uint4*>(g_qd_masks)[x];
  m0 = ((uint64_t)mm.y << 32) | mm.x;
  m1 = ((uint64_t)mm.w << 32) | mm.z;
}

// Occ for lo and hi of one backward step, all gathers issued before any is used.  lo and hi
// often share a line ("cache lines are automatically reused"); then the line's
// sectors and the superblock word are loaded once and reused from registers, which halves the
// L1 wavefronts of a step when the structure is L2-resident.  N < 2^32: u32 arithmetic.
template <int SMS = 0, bool MT = false>   // MT: masks from the per-CTA table (qd_masks_init)
__device__ __forceinline__ void fm_step16(const FmParams& F, uint32_t c, uint32_t& lo, uint32_t& hi, uint32_t& lines) {
  uint32_t jl = (lo >> 5) / 7u;                                  // floor(lo/224)
  uint32_t jh = (hi >> 5) / 7u;
  jl = jl > (uint32_t)F.last_line ? (uint32_t)F.last_line : jl;
  jh = jh > (uint32_t)F.last_line ? (uint32_t)F.last_line : jh;
  const uint32_t pl = 32u + lo - jl * (uint32_t)QD_B, ph = 32u + hi - jh * (uint32_t)QD_B;
  const bool same = jl == jh;
  const bool rl_ = pl >= 128, rh_ = ph >= 128;
  uint64_t al[4], bl[4] = {0, 0, 0, 0}, ah[4] = {0, 0, 0, 0}, bh[4] = {0, 0, 0, 0};
  const uint4* Ll = F.lines + 4 * (uint64_t)jl;
  const uint4* Lh = F.lines + 4 * (uint64_t)jh;
  ld_sector(Ll, al[0], al[1], al[2], al[3]);
  if (rl_) ld_sector(Ll + 2, bl[0], bl[1], bl[2], bl[3]);
  if (!same) ld_sector(Lh, ah[0], ah[1], ah[2], ah[3]);
  if (rh_ && !(same && rl_)) ld_sector(Lh + 2, bh[0], bh[1], bh[2], bh[3]);
  const uint32_t sl = fm_super<SMS>(F, jl >> QD_SB_LOG, c);
  const bool same_sb = (jl >> QD_SB_LOG) == (jh >> QD_SB_LOG);
  uint32_t sh = same_sb ? sl : fm_super<SMS>(F, jh >> QD_SB_LOG, c);
  if (same) {
#pragma unroll
    for (int t = 0; t < 4; ++t) ah[t] = al[t];
    if (rl_) {
#pragma unroll
      for (int t = 0; t < 4; ++t) bh[t] = bl[t];
    }
  }
  lines = same ? 1u : 2u;
  const uint64_t cl = 0ull - (uint64_t)(c & 1u), ch = 0ull - (uint64_t)(c >> 1);
  auto rank1 = [&](const uint64_t* a, const uint64_t* b, uint32_t p, uint32_t s) -> uint32_t {
    const bool right = p >= 128;
    const int x = (int)(p & 127u);
    const uint64_t inv = right ? 0ull : ~0ull;
    const uint64_t* w = right ? b : a;
    uint64_t m0, m1;
    if (MT) qd_masks((uint32_t)x, m0, m1);
    else { m0 = prefix_mask(x, 0); m1 = prefix_mask(x, 1); }
    uint32_t cnt = __popcll((w[0] ^ cl) & (w[1] ^ ch) & (m0 ^ inv)) +
                   __popcll((w[2] ^ cl) & (w[3] ^ ch) & (m1 ^ inv));
    uint64_t dw = (c & 2u) ? a[1] : a[0];
    uint32_t base = (s << QD_SHIFT) + (uint32_t)((dw >> (16 * (c & 1u))) & 0xffffull);
    return right ? base + cnt : base - cnt;
  };
  uint32_t rl = rank1(al, bl, pl, sl), rh = rank1(ah, bh, ph, sh);
  // '$' is stored as A at row spos: Occ(A, x) = rank(x, A) - [x > spos]
  if (c == 0) { rl -= (lo > (uint32_t)F.spos); rh -= (hi > (uint32_t)F.spos); }
  const uint32_t Cc = __ldg(F.Ct + c);   // L1-resident; a register-indexed param array costs ~26 SASS
  lo = Cc + rl;
  hi = Cc + rh;
}

// ---- the same step over a QuadRank16x2 BWT (variants.cu, reading R25): every rank reads one
// 32-B sector (four u16 deltas to the sector's char 48 + 96 packed chars); lo and hi share the
// load when they fall in the same sector.  Superblock words as QuadRank16 (fm_super).
__device__ __forceinline__ void x2_locate(uint32_t x, uint32_t last_line, uint32_t& j, uint32_t& h, uint32_t& p) {
  uint32_t jj = (x >> 6) / 3u;                                    // floor(x/192)
  jj = jj > last_line ? last_line : jj;
  uint32_t d = x - jj * (uint32_t)Q16X2_B;
  d = d > (uint32_t)Q16X2_B - 1 ? (uint32_t)Q16X2_B - 1 : d;
  h = d >= 96 ? 1u : 0u;
  p = d - 96u * h;
  j = jj;
}
// count of symbol c among the sector's chars between p and its anchor 48, signed by the side
// The two count masks of every in-sector position p (0..95), built once per CTA in shared memory
// by kernels over a QuadRank16x2 BWT (x2_masks_init): one 16-B shared load per rank instead of
// the variable 64-bit shifts of two prefix masks (that kernel is issue-bound, ncu).
__shared__ __align__(16) uint64_t g_x2_masks[96][2];

__device__ __forceinline__ uint64_t x2_range_calc(uint32_t p, int t);
__device__ __forceinline__ void x2_masks_init() {
  for (uint32_t i = threadIdx.x; i < 96; i += blockDim.x) {
    g_x2_masks[i][0] = x2_range_calc(i, 0);
    g_x2_masks[i][1] = x2_range_calc(i, 1);
  }
  __syncthreads();
}
__device__ __forceinline__ uint64_t x2_range_calc(uint32_t p, int t) {
  return (prefix_mask((int)p, t) ^ prefix_mask(48, t)) & (t ? 0xffffffffull : ~0ull);
}
__device__ __forceinline__ uint32_t x2_rank(const uint64_t (&w)[4], uint32_t p, uint32_t c, uint32_t s) {
  const uint64_t nl = (c & 1u) ? 0ull : ~0ull, nh = (c & 2u) ? 0ull : ~0ull;   // planes (variants.cu)
  const uint4 mm = reinterpret_cast<const uint4*>(g_x2_masks)[p];
  const uint64_t m0 = ((uint64_t)mm.y << 32) | mm.x, m1 = ((uint64_t)mm.w << 32) | mm.z;
  const uint32_t cnt = __popcll((w[1] ^ nl) & (w[2] ^ nh) & m0) +
                       __popcll((w[3] ^ nl) & ((w[3] >> 32) ^ nh) & m1);
  const uint32_t base = (s << QD_SHIFT) + (uint32_t)((w[0] >> (16 * c)) & 0xffffull);
  return p >= 48 ? base + cnt : base - cnt;
}

template <int SMS = 0>
__device__ __forceinline__ void fm_step_x2(const FmParams& F, uint32_t c, uint32_t& lo, uint32_t& hi, uint32_t& lines,
                                           const uint4* C4 = nullptr) {
  uint32_t jl, hl, pl, jh, hh, ph;
  x2_locate(lo, (uint32_t)F.last_line, jl, hl, pl);
  x2_locate(hi, (uint32_t)F.last_line, jh, hh, ph);
  const bool same = jl == jh && hl == hh;
  uint64_t a[4], b[4] = {0, 0, 0, 0};
  ld_sector(F.lines + 4 * (uint64_t)jl + 2 * hl, a[0], a[1], a[2], a[3]);
  if (!same) ld_sector(F.lines + 4 * (uint64_t)jh + 2 * hh, b[0], b[1], b[2], b[3]);
  const uint32_t sl = fm_super<SMS>(F, jl >> QD_SB_LOG, c);
  const uint32_t sh = (jl >> QD_SB_LOG) == (jh >> QD_SB_LOG) ? sl : fm_super<SMS>(F, jh >> QD_SB_LOG, c);
  if (same) {
#pragma unroll
    for (int t = 0; t < 4; ++t) b[t] = a[t];
  }
  lines = jl == jh ? 1u : 2u;
  uint32_t rl = x2_rank(a, pl, c, sl), rh = x2_rank(b, ph, c, sh);
  if (c == 0) { rl -= (lo > (uint32_t)F.spos); rh -= (hi > (uint32_t)F.spos); }
  // C[c] from registers when the caller holds them (select, no load on the step's critical path)
  const uint32_t Cc = C4 ? (c & 2u ? (c & 1u ? C4->w : C4->z) : (c & 1u ? C4->y : C4->x)) : __ldg(F.Ct + c);
  lo = Cc + rl;
  hi = Cc + rh;
}

// one backward step over either BWT layout (BW 0: QuadRank16 de-duplicating step, 1: QuadRank16x2)
template <int SMS = 0, int BW = 0, bool MT = false>
__device__ __forceinline__ void fm_step(const FmParams& F, uint32_t c, uint32_t& lo, uint32_t& hi, uint32_t& lines) {
  if (BW == 1) fm_step_x2<SMS>(F, c, lo, hi, lines);
  else         fm_step16<SMS, MT>(F, c, lo, hi, lines);
}

// The exact step of the approximate-search continuations: when lo and hi fall in one half line
// (QuadRank16) or one sector (QuadRank16x2) — nearly always, the intervals there being narrow —
// both ranks come from one gather, one delta, one superblock word and one C[c], Occ(c, hi)
// differing from Occ(c, lo) only in the count mask; otherwise the general step.
template <int BW>
__device__ __forceinline__ void fm_step_cont(const FmParams& F, uint32_t c, uint32_t& lo, uint32_t& hi,
                                             uint32_t& lines) {
  if (BW == 0) {
    const uint32_t j = (lo >> 5) / 7u, jh = (hi >> 5) / 7u;          // lo, hi <= N: j <= last_line
    const uint32_t pl = lo + 32u - j * (uint32_t)QD_B, ph = hi + 32u - j * (uint32_t)QD_B;
    const bool rx = pl >= 128u;
    if (jh == j && (ph >= 128u) == rx) {
      const uint64_t* L = reinterpret_cast<const uint64_t*>(F.lines) + 8 * (uint64_t)j;
      uint64_t a0, a1, a2, a3;
      ld_sector(L + (rx ? 4 : 0), a0, a1, a2, a3);
      const uint64_t dr = ldg_u64_if(rx, L + (c >> 1));
      const uint32_t sv = __ldg(F.super + 4 * (j >> QD_SB_LOG) + c);
      const uint64_t cl = 0ull - (uint64_t)(c & 1u), ch = 0ull - (uint64_t)(c >> 1);
      const uint64_t ma0 = (a0 ^ cl) & (a1 ^ ch), ma1 = (a2 ^ cl) & (a3 ^ ch);
      const uint64_t inv = rx ? ~0ull : 0ull;
      const uint32_t xx = pl & 127u, yy = ph & 127u;
      const uint32_t d0 = min(xx, 64u), d1 = xx - d0, e0 = min(yy, 64u), e1 = yy - e0;
      const uint32_t cx = __popcll(ma0 & (ones_shl(d0) ^ inv)) + __popcll(ma1 & (ones_shl(d1) ^ inv));
      const uint32_t cy = __popcll(ma0 & (ones_shl(e0) ^ inv)) + __popcll(ma1 & (ones_shl(e1) ^ inv));
      const uint64_t dw = rx ? dr : ((c & 2u) ? a1 : a0);
      const uint32_t base = (sv << QD_SHIFT) + (uint32_t)((dw >> (16 * (c & 1u))) & 0xffffull);
      const uint32_t dol = c == 0 ? 1u : 0u;
      const uint32_t vx = (rx ? base + cx : base - cx) - (dol & (lo > (uint32_t)F.spos ? 1u : 0u));
      const uint32_t vy = (rx ? base + cy : base - cy) - (dol & (hi > (uint32_t)F.spos ? 1u : 0u));
      const uint32_t Cc = __ldg(F.Ct + c);
      lo = Cc + vx;
      hi = Cc + vy;
      lines = 1;
      return;
    }
    fm_step16<0, false>(F, c, lo, hi, lines);             // arithmetic masks: no shared table needed
  } else {
    uint32_t j, h, p, jh, hh, ph;
    x2_locate(lo, (uint32_t)F.last_line, j, h, p);
    x2_locate(hi, (uint32_t)F.last_line, jh, hh, ph);
    if (jh == j && hh == h) {
      uint64_t w0, w1, w2, w3;
      ld_sector(F.lines + 4 * (uint64_t)j + 2 * h, w0, w1, w2, w3);
      const uint32_t sv = __ldg(F.super + 4 * (j >> QD_SB_LOG) + c);
      const uint64_t nl = (c & 1u) ? 0ull : ~0ull, nh = (c & 2u) ? 0ull : ~0ull;
      const uint64_t m0 = (w1 ^ nl) & (w2 ^ nh);
      const uint32_t m1 = ((uint32_t)w3 ^ (uint32_t)nl) & ((uint32_t)(w3 >> 32) ^ (uint32_t)nh);
      const uint4 mx = reinterpret_cast<const uint4*>(g_x2_masks)[p];
      const uint4 my = reinterpret_cast<const uint4*>(g_x2_masks)[ph];
      const uint32_t cx = __popcll(m0 & (((uint64_t)mx.y << 32) | mx.x)) + __popc(m1 & mx.z);
      const uint32_t cy = __popcll(m0 & (((uint64_t)my.y << 32) | my.x)) + __popc(m1 & my.z);
      const uint32_t base = (sv << QD_SHIFT) + (uint32_t)((w0 >> (16 * c)) & 0xffffull);
      const uint32_t dol = c == 0 ? 1u : 0u;
      const uint32_t vx = (p >= 48 ? base + cx : base - cx) - (dol & (lo > (uint32_t)F.spos ? 1u : 0u));
      const uint32_t vy = (ph >= 48 ? base + cy : base - cy) - (dol & (hi > (uint32_t)F.spos ? 1u : 0u));
      const uint32_t Cc = __ldg(F.Ct + c);
      lo = Cc + vx;
      hi = Cc + vy;
      lines = 1;
      return;
    }
    fm_step_x2<0>(F, c, lo, hi, lines);
  }
}

template <int BW>
__global__ void k_kmer_table(FmParams F, uint2* __restrict__ table) {
  if (BW == 1) x2_masks_init();
  else qd_masks_init();
  const uint32_t key = blockIdx.x * blockDim.x + threadIdx.x;
  if (key >= (1u << (2 * F.K))) return;
  uint32_t lo = 0, hi = (uint32_t)F.N;
  uint32_t dummy;
  for (int t = 0; t < F.K && lo < hi; ++t) fm_step<0, BW, true>(F, (key >> (2 * t)) & 3u, lo, hi, dummy);   // last char first
  if (lo >= hi) lo = hi = 0;
  table[key] = make_uint2(lo, hi);
}

// Pattern symbols are read through an 8-byte window held in a register (one aligned u64
// load per 8 steps instead of one byte load per step: a warp's 32 lanes read 32 different
// patterns, so every load instruction costs 32 L1 wavefronts).
struct PatWindow {
  const uint8_t* base;
  uint64_t word;
  int64_t wk;        // index (relative to base's aligned start) of the cached word, -1 if none
  uint32_t mis;      // base misalignment in bytes
  __device__ __forceinline__ void reset(const uint8_t* P) {
    mis = (uint32_t)((uintptr_t)P & 7u);
    base = P - mis;
    wk = -1;
  }
  // The reload is a predicated load every lane issues (no branch), so a warp whose lanes cross
  // their 8-byte windows at different steps does not split (ncu: the branchy reload ran with ~2
  // of 32 lanes active in every loop iteration of the count kernel).
  // at() for lanes that may hold no task (act == false): no load is issued for them
  __device__ __forceinline__ uint32_t at_if(bool act, int64_t k) {
    const int64_t a = k + mis;
    const int64_t w = a >> 3;
    const bool need = act && w != wk;
    ldg_u64_keep(need, reinterpret_cast<const unsigned long long*>(base) + w, word);
    wk = need ? w : wk;
    return (uint32_t)(word >> (8 * ((uint32_t)a & 7u))) & 3u;
  }
  __device__ __forceinline__ uint32_t at(int64_t k) {
    const int64_t a = k + mis;
    const int64_t w = a >> 3;
    const bool need = w != wk;
    ldg_u64_keep(need, reinterpret_cast<const unsigned long long*>(base) + w, word);
    wk = w;
    return (uint32_t)(word >> (8 * ((uint32_t)a & 7u))) & 3u;
  }
};

// Lean variant of fm_step (knob "fm_step" = 1): each rank loads its counted half directly
// (sector 0 left of the anchor, sector 1 right of it) and, only when right, the one u64 word of
// sector 0 that holds its delta; no de-duplication of shared lines (the L1 merges them), so no
// register copies or half selects.  Fewer instructions, a few more L1 wavefronts.
__device__ __forceinline__ uint32_t fm_rank_lean(const FmParams& F, uint32_t j, uint32_t p, uint32_t c, uint64_t cl,
                                                 uint64_t ch, uint32_t s) {
  const bool right = p >= 128;
  const uint4* L = F.lines + 4 * (uint64_t)j;
  uint64_t w0, w1, w2, w3;
  ld_sector(L + 2 * (right ? 1 : 0), w0, w1, w2, w3);
  uint64_t dr = 0;
  if (right) dr = __ldg(reinterpret_cast<const unsigned long long*>(L) + (c >> 1));
  const int xx = (int)(p & 127u);
  const uint64_t inv = right ? 0ull : ~0ull;
  const uint32_t cnt = __popcll((w0 ^ cl) & (w1 ^ ch) & (prefix_mask(xx, 0) ^ inv)) +
                       __popcll((w2 ^ cl) & (w3 ^ ch) & (prefix_mask(xx, 1) ^ inv));
  const uint64_t dw = right ? dr : ((c & 2u) ? w1 : w0);
  const uint32_t base = (s << QD_SHIFT) + (uint32_t)((dw >> (16 * (c & 1u))) & 0xffffull);
  return right ? base + cnt : base - cnt;
}

// C[c] from four registers (3 selects) instead of an L1 load: the lean step is L1-bound on an
// L2-resident BWT (ncu: L1 91% busy), so ALU is the cheaper resource.
__device__ __forceinline__ uint32_t pick4(uint4 v, uint32_t c) {
  return (c & 2u) ? ((c & 1u) ? v.w : v.z) : ((c & 1u) ? v.y : v.x);
}

template <int SMS>
__device__ __forceinline__ void fm_step_lean(const FmParams& F, uint4 C4, uint32_t c, uint32_t& lo, uint32_t& hi,
                                             uint32_t& lines) {
  const uint64_t cl = 0ull - (uint64_t)(c & 1u), ch = 0ull - (uint64_t)(c >> 1);
  const uint32_t jl = (lo >> 5) / 7u, jh = (hi >> 5) / 7u;   // lo, hi <= N: j <= last_line
  const uint32_t pl = 32u + lo - jl * (uint32_t)QD_B, ph = 32u + hi - jh * (uint32_t)QD_B;
  // one superblock-word load when both ranks fall in the same superblock (nearly always)
  const uint32_t sl = fm_super<SMS>(F, jl >> QD_SB_LOG, c);
  const uint32_t sh = (jl >> QD_SB_LOG) == (jh >> QD_SB_LOG) ? sl : fm_super<SMS>(F, jh >> QD_SB_LOG, c);
  uint32_t rl = fm_rank_lean(F, jl, pl, c, cl, ch, sl);
  uint32_t rh = fm_rank_lean(F, jh, ph, c, cl, ch, sh);
  lines = jl == jh ? 1u : 2u;
  if (c == 0) { rl -= (lo > (uint32_t)F.spos); rh -= (hi > (uint32_t)F.spos); }
  const uint32_t Cc = pick4(C4, c);
  lo = Cc + rl;
  hi = Cc + rh;
}

// ---- the "one line per iteration" step (knob fm_step = 3; default on L2-resident BWTs) -------
// A backward step ranks c at lo and at hi.  After the k-mer seed the interval
// is narrow, so lo and hi nearly always fall in one line ("cache lines are
// automatically reused"); then one line gather, one delta, one superblock word and one C[c]
// serve both ranks, and Occ(c, hi) differs from Occ(c, lo) only by the masked popcount of that
// line's own planes.  When they do not share a line, the step takes two loop iterations: this
// one ranks at lo (`pend` set, hi kept), the next ranks at hi.  Every iteration therefore runs
// the same instructions — one line, up to two masked counts — and no lane of a warp waits on a
// divergent second-rank path.  Returns true when the step is complete.
__device__ __forceinline__ uint64_t half_mask(uint32_t xx, int t, bool right) {
  // chars [xx, 128) of a half (left of the anchor) or [0, xx) (right of it), word t (64 chars)
  const uint64_t pm = prefix_mask((int)xx, t);
  return right ? pm : ~pm;
}

template <int SMS>
__device__ __forceinline__ bool fm_step_pend(const FmParams& F, uint4 C4, uint32_t c, uint32_t& lo, uint32_t& hi,
                                             uint32_t& pend, uint32_t& lines) {
  const uint32_t x = pend ? hi : lo;
  const uint32_t j = (x >> 5) / 7u;                    // floor(x / 224); lo, hi <= N: j <= last_line
  const uint32_t jy = (hi >> 5) / 7u;
  const uint32_t p = x + 32u - j * (uint32_t)QD_B;
  const uint32_t py = hi + 32u - j * (uint32_t)QD_B;   // meaningful when jy == j
  const bool rx = p >= 128u;
  // hi is ranked in this iteration when it lies in the same half line (same 32-B sector, same
  // delta); a pair split by the anchor or by a line boundary takes a second iteration
  const bool two = !pend && jy == j && ((py >= 128u) == rx);
  lines = pend ? 0u : (jy == j ? 1u : 2u);             // distinct lines of the step, counted once
  const uint64_t* L = reinterpret_cast<const uint64_t*>(F.lines) + 8 * (uint64_t)j;
  uint64_t a0, a1, a2, a3;
  ld_sector(L + (rx ? 4 : 0), a0, a1, a2, a3);
  const uint64_t dr = ldg_u64_if(rx, L + (c >> 1));   // right of the anchor: the delta word of sector 0
  const uint32_t s = fm_super<SMS>(F, j >> QD_SB_LOG, c);
  const uint64_t cl = 0ull - (uint64_t)(c & 1u), ch = 0ull - (uint64_t)(c >> 1);
  const uint64_t ma0 = (a0 ^ cl) & (a1 ^ ch), ma1 = (a2 ^ cl) & (a3 ^ ch);   // c at each char of the half
  // count masks: left of the anchor chars [xx, 128) = ~0 << d_t per word; right chars [0, xx) = its complement
  const uint64_t inv = rx ? ~0ull : 0ull;
  const uint32_t xx = p & 127u, yy = py & 127u;
  const uint32_t d0 = min(xx, 64u), d1 = xx - d0, e0 = min(yy, 64u), e1 = yy - e0;
  const uint32_t cx = __popcll(ma0 & (ones_shl(d0) ^ inv)) + __popcll(ma1 & (ones_shl(d1) ^ inv));
  const uint32_t cy = __popcll(ma0 & (ones_shl(e0) ^ inv)) + __popcll(ma1 & (ones_shl(e1) ^ inv));
  const uint64_t dw = rx ? dr : ((c & 2u) ? a1 : a0);
  const uint32_t base = (s << QD_SHIFT) + (uint32_t)((dw >> (16 * (c & 1u))) & 0xffffull);
  const uint32_t dol = c == 0 ? 1u : 0u;               // '$' stored as A at row spos
  const uint32_t vx = (rx ? base + cx : base - cx) - (dol & (x > (uint32_t)F.spos ? 1u : 0u));
  const uint32_t vy = (rx ? base + cy : base - cy) - (dol & (hi > (uint32_t)F.spos ? 1u : 0u));
  const uint32_t Cc = pick4(C4, c);
  const uint32_t nlo = Cc + vx, nhi = Cc + vy;
  const bool done = pend || two;
  lo = pend ? lo : nlo;
  hi = pend ? nlo : (two ? nhi : hi);
  pend = done ? 0u : 1u;
  return done;
}

// The same over a QuadRank16x2 BWT: lo and hi share the iteration when they fall in one 32-B
// sector (one gather, one delta, one superblock word); otherwise two iterations.
template <int SMS>
__device__ __forceinline__ bool fm_step_pend_x2(const FmParams& F, uint4 C4, uint32_t c, uint32_t& lo, uint32_t& hi,
                                                uint32_t& pend, uint32_t& lines) {
  const uint32_t x = pend ? hi : lo;
  uint32_t j, h, p, jy, hy, py;
  x2_locate(x, (uint32_t)F.last_line, j, h, p);
  x2_locate(hi, (uint32_t)F.last_line, jy, hy, py);
  const bool two = !pend && jy == j && hy == h;
  lines = pend ? 0u : (jy == j ? 1u : 2u);
  uint64_t w0, w1, w2, w3;
  ld_sector(F.lines + 4 * (uint64_t)j + 2 * h, w0, w1, w2, w3);
  const uint32_t s = fm_super<SMS>(F, j >> QD_SB_LOG, c);
  const uint64_t nl = (c & 1u) ? 0ull : ~0ull, nh = (c & 2u) ? 0ull : ~0ull;   // planes (variants.cu)
  const uint64_t m0 = (w1 ^ nl) & (w2 ^ nh);
  const uint32_t m1 = ((uint32_t)w3 ^ (uint32_t)nl) & ((uint32_t)(w3 >> 32) ^ (uint32_t)nh);
  const uint4 mx = reinterpret_cast<const uint4*>(g_x2_masks)[p];
  const uint4 my = reinterpret_cast<const uint4*>(g_x2_masks)[two ? py : p];
  const uint32_t cx = __popcll(m0 & (((uint64_t)mx.y << 32) | mx.x)) + __popc(m1 & mx.z);
  const uint32_t cy = __popcll(m0 & (((uint64_t)my.y << 32) | my.x)) + __popc(m1 & my.z);
  const uint32_t base = (s << QD_SHIFT) + (uint32_t)((w0 >> (16 * c)) & 0xffffull);
  const uint32_t dol = c == 0 ? 1u : 0u;
  const uint32_t vx = (p >= 48 ? base + cx : base - cx) - (dol & (x > (uint32_t)F.spos ? 1u : 0u));
  const uint32_t vy = (py >= 48 ? base + cy : base - cy) - (dol & (hi > (uint32_t)F.spos ? 1u : 0u));
  const uint32_t Cc = pick4(C4, c);
  const uint32_t nlo = Cc + vx, nhi = Cc + vy;
  const bool done = pend || two;
  lo = pend ? lo : nlo;
  hi = pend ? nlo : (two ? nhi : hi);
  pend = done ? 0u : 1u;
  return done;
}

// 8-mer table key of the pattern's last 8 symbols (P[len-8..len), 2 bits each, the last symbol
// in the low bits — PAPER.md:918, reading R14) from one unaligned 8-byte read: reverse the byte
// order, keep 2 bits per byte and compact the eight 2-bit fields into 16 bits.
__device__ __forceinline__ uint64_t load8_unaligned(const uint8_t* p) {
  const uintptr_t a = (uintptr_t)p;
  const unsigned long long* base = reinterpret_cast<const unsigned long long*>(a & ~(uintptr_t)7);
  const uint32_t sh = (uint32_t)(a & 7u) * 8u;
  uint64_t x = __ldg(base);
  if (sh) x = (x >> sh) | ((uint64_t)__ldg(base + 1) << (64u - sh));
  return x & 0x0303030303030303ull;
}
// compact the 2-bit fields at bits 8t (t = 0..7) to bits 2t
__device__ __forceinline__ uint32_t compact8(uint64_t r) {
  r = (r | (r >> 6)) & 0x000F000F000F000Full;
  r = (r | (r >> 12)) & 0x000000FF000000FFull;
  r = (r | (r >> 24)) & 0xFFFFull;
  return (uint32_t)r;
}
__device__ __forceinline__ uint32_t kmer_key8(const uint8_t* last8) {
  uint64_t x = load8_unaligned(last8);
  return compact8(((uint64_t)__byte_perm((uint32_t)x, 0, 0x0123) << 32) | __byte_perm((uint32_t)(x >> 32), 0, 0x0123));
}
// Key of the reverse complement's last 8 symbols: RC(P)[len-1-t] = 3 - P[t], so the key is
// sum_t (3 - P[t]) << 2t = 0xFFFF ^ (P[0..8) compacted without byte reversal).
__device__ __forceinline__ uint32_t kmer_key8_rc(const uint8_t* first8) { return 0xFFFFu ^ compact8(load8_unaligned(first8)); }

// STRANDS = 1: count each pattern as given.  STRANDS = 2: task 2i counts pattern i and task
// 2i+1 its reverse complement RC(P)[j] = 3 - P[len-1-j] ("both forward and
// reverse-complement direction"; NEXT §8(f)1), read from the same bytes in the opposite
// direction, so no reverse-complemented copy is ever materialised.
// Table key of width K (<= 12) of the pattern's last K symbols: sum_{t<K} P[len-1-t] << 2t.
// K = 8 (the paper's table) is one unaligned 8-byte read; other widths read symbol by symbol
// through the pattern window (no read before the pattern's first byte).
__device__ __forceinline__ uint32_t kmer_key(int K, PatWindow& P, const uint8_t* p, uint32_t len) {
  if (K == 8) return kmer_key8(p + len - 8);
  if (K > 8 && len >= 16) {
    // P[len-K .. len-8) are the last K-8 bytes of the 8 bytes ending at len-8 (no read before p)
    const uint32_t hi8 = kmer_key8(p + len - 16) & ((1u << (2 * (K - 8))) - 1u);
    return kmer_key8(p + len - 8) | (hi8 << 16);
  }
  uint32_t key = 0;
  for (int t = 0; t < K; ++t) key |= P.at((int64_t)len - 1 - t) << (2 * t);
  return key;
}
// Reverse-complement key: sum_{t<K} (3 - P[t]) << 2t.
__device__ __forceinline__ uint32_t kmer_key_rc(int K, PatWindow& P, const uint8_t* p, uint32_t len) {
  if (K == 8) return kmer_key8_rc(p);
  if (K > 8 && len >= 16) return kmer_key8_rc(p) | ((kmer_key8_rc(p + 8) & ((1u << (2 * (K - 8))) - 1u)) << 16);
  uint32_t key = 0;
  for (int t = 0; t < K; ++t) key |= (3u - P.at(t)) << (2 * t);
  return key;
}

// Pattern symbols of one strand for the approximate-search kernels: STRANDS = 2 tasks with rc = 1
// read the reverse complement RC(P)[k] = 3 - P[len-1-k] from the same bytes.
template <int STRANDS>
struct StrandWindow {
  PatWindow P;
  uint32_t len, rc;
  __device__ __forceinline__ void reset(const uint8_t* p, uint32_t l, uint32_t r) { P.reset(p); len = l; rc = r; }
  __device__ __forceinline__ uint32_t at(int64_t k) {
    if (STRANDS == 1) return P.at(k);
    return rc ? 3u - P.at((int64_t)len - 1 - k) : P.at(k);
  }
};

// 4 resident CTAs (64 registers): capping registers for 6 or 8 CTAs/SM spills and runs 2-4x
// slower on configs[3]/[4] (profiles/r01_fm_occupancy_sweep.jsonl).
// Seed pre-pass of the dynamic-order count kernel: one thread per task computes the k-mer table
// interval of its (virtual) pattern — the key of the last K symbols, or of the reverse
// complement's, and one table lookup — fully in parallel, so that the search loop's refill path
// is a single 8-byte load.  Inline seeding ran in ~94% of the loop iterations with ~3 of 32
// lanes active and cost ~40% of the kernel's instructions (ncu source page, configs[3]).
template <bool FIXED, int STRANDS>
__global__ void __launch_bounds__(256) k_fm_seed(FmParams F, const uint8_t* __restrict__ pat,
                                                 const uint64_t* __restrict__ offs, const uint32_t* __restrict__ lens,
                                                 uint32_t fixed_len, uint64_t m, uint2* __restrict__ seeds) {
  const uint64_t ntask = m * STRANDS;
  for (uint64_t ti = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ti < ntask; ti += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pi = STRANDS == 2 ? ti >> 1 : ti;
    const uint32_t rc = STRANDS == 2 ? (uint32_t)(ti & 1) : 0u;
    const uint32_t len = FIXED ? fixed_len : lens[pi];
    const uint8_t* p = pat + (FIXED ? pi * (uint64_t)fixed_len : offs[pi]);
    uint2 iv = make_uint2(0u, (uint32_t)F.N);
    if (F.K && len >= (uint32_t)F.K) {
      PatWindow P;
      P.reset(p);
      iv = __ldg(F.kmer + (rc ? kmer_key_rc(F.K, P, p, len) : kmer_key(F.K, P, p, len)));
    }
    seeds[ti] = iv;
  }
}

// Seed pre-pass of k_fm_count_l2 for fixed-length batches whose post-seed part has <= 32
// symbols (configs[3]: 32 - 12 = 20): besides the k-mer interval it packs the symbols the
// backward search will consume, in consumption order, 2 bits each (bits [2t, 2t+2) = the t-th
// step's symbol; reverse-complemented for STRANDS = 2 odd tasks).  The count kernel then takes
// each step's symbol from a register shift instead of an 8-byte pattern window (address
// arithmetic and a predicated load per step), and never reads the pattern bytes.
// 2-bit fields of a 128-bit word in reverse order (field i -> field 63 - i)
__device__ __forceinline__ unsigned __int128 rev2_128(unsigned __int128 a) {
  const uint64_t lo = (uint64_t)a, hi = (uint64_t)(a >> 64);
  auto rev2 = [](uint64_t x) {
    x = __brevll(x);
    return ((x >> 1) & 0x5555555555555555ull) | ((x & 0x5555555555555555ull) << 1);
  };
  return ((unsigned __int128)rev2(lo) << 64) | rev2(hi);
}

template <int STRANDS>
__global__ void __launch_bounds__(256) k_fm_seed_packed(FmParams F, const uint8_t* __restrict__ pat, uint32_t len,
                                                        uint64_t m, uint4* __restrict__ seeds) {
  const uint64_t ntask = m * STRANDS;
  const uint32_t kused = (F.K && len >= (uint32_t)F.K) ? (uint32_t)F.K : 0u;
  const uint32_t nrem = len - kused;                       // <= 32 (checked by the launcher); len <= 46
  const unsigned __int128 one = 1;
  for (uint64_t ti = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ti < ntask; ti += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pi = STRANDS == 2 ? ti >> 1 : ti;
    const uint32_t rc = STRANDS == 2 ? (uint32_t)(ti & 1) : 0u;
    const uint8_t* p = pat + pi * (uint64_t)len;
    // A = the pattern's symbols 2 bits each, P[i] at bits [2i, 2i+2), from the aligned 8-byte
    // words covering [p, p + len) (<= 7 words: 53 bytes)
    const uint32_t mis = (uint32_t)((uintptr_t)p & 7u);
    const unsigned long long* w = reinterpret_cast<const unsigned long long*>(p - mis);
    const uint32_t nw = (mis + len + 7) >> 3;
    unsigned __int128 A = 0;
    for (uint32_t i = 0; i < nw; ++i) A |= (unsigned __int128)compact8(__ldg(w + i) & 0x0303030303030303ull) << (16 * i);
    A >>= 2 * mis;
    const unsigned __int128 R = rev2_128(A);               // P[i] at bits [126 - 2i, 128 - 2i)
    uint2 iv = make_uint2(0u, (uint32_t)F.N);
    uint64_t sy;
    if (rc) {   // RC(P)[j] = 3 - P[len-1-j]: key over its last K = sum_t (3 - P[t]) << 2t
      if (kused) iv = __ldg(F.kmer + (uint32_t)((A ^ ((one << (2 * kused)) - 1)) & ((one << (2 * kused)) - 1)));
      sy = (uint64_t)(((A >> (2 * kused)) ^ ((one << (2 * nrem)) - 1)) & ((one << (2 * nrem)) - 1));
    } else {    // key = sum_t P[len-1-t] << 2t; symbols P[nrem-1], P[nrem-2], ..., P[0]
      if (kused) iv = __ldg(F.kmer + (uint32_t)((R >> (128 - 2 * len)) & ((one << (2 * kused)) - 1)));
      sy = nrem ? (uint64_t)((R >> (128 - 2 * nrem)) & ((one << (2 * nrem)) - 1)) : 0ull;
    }
    seeds[ti] = make_uint4(iv.x, iv.y, (uint32_t)sy, (uint32_t)(sy >> 32));
  }
}

// Work order.  DYN = false: the lane's own grid-stride task sequence (ti, ti + stride, ...) over
// a multi-wave grid.  DYN = true (default): a persistent grid whose warps take chunks of
// FM_CHUNK tasks from a global counter (one atomicAdd per chunk); in every loop iteration the
// lanes that finished a pattern are handed the chunk's next tasks by their rank in a ballot, so
// a warp keeps all 32 lanes busy until the whole batch is drained.  With the static order a
// lane had ~4 patterns of very different lengths (exact vs random, 24 vs 6 steps) and warps ran
// with 19 of 32 lanes active on average (ncu source page, profiles/r01_ncu_cluster.md capture).
constexpr uint32_t FM_CHUNK = 64;
#ifndef QR_FM_MINB
#define QR_FM_MINB 4
#endif

template <bool FIXED, bool WORK, int STRANDS, int STEP, int SMS, bool DYN, int BW = 0>
__global__ void __launch_bounds__(256, QR_FM_MINB) k_fm_count(FmParams F, const uint8_t* __restrict__ pat,
                                                     const uint64_t* __restrict__ offs, const uint32_t* __restrict__ lens,
                                                     uint32_t fixed_len, uint32_t* __restrict__ out,
                                                     uint32_t* __restrict__ out_rc, uint64_t m,
                                                     unsigned long long* __restrict__ work,
                                                     unsigned long long* __restrict__ ctr,
                                                     const uint2* __restrict__ seeds) {
  if (BW == 1) x2_masks_init();
  fm_preload_super<SMS>(F);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t ntask = m * STRANDS;
  const uint4 C4 = __ldg(reinterpret_cast<const uint4*>(F.Ct));
  uint64_t ti = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t lo = 0, hi = 0, len = 0, rc = 0;
  int64_t k = -1;
  PatWindow P;
  uint64_t n_steps = 0, n_lines = 0;
  // seed task ti: the 8-mer table interval of the (virtual) pattern's last 8 symbols, or [0, N)
  auto seed = [&]() {
    const uint64_t pi = STRANDS == 2 ? ti >> 1 : ti;
    rc = STRANDS == 2 ? (uint32_t)(ti & 1) : 0u;
    len = FIXED ? fixed_len : lens[pi];
    const uint8_t* p = pat + (FIXED ? pi * (uint64_t)fixed_len : offs[pi]);
    P.reset(p);
    const bool tab = F.K && len >= (uint32_t)F.K;
    uint2 iv;
    if (DYN && seeds) iv = __ldg(seeds + ti);             // precomputed by k_fm_seed
    else iv = tab ? __ldg(F.kmer + (rc ? kmer_key_rc(F.K, P, p, len) : kmer_key(F.K, P, p, len)))
                  : make_uint2(0u, (uint32_t)F.N);
    lo = iv.x; hi = iv.y;
    k = (int64_t)len - 1 - (tab ? F.K : 0);
    // issue the load of the first searched symbol's word now, so that it overlaps the seed load
    // instead of following it (the first step's symbol is otherwise a dependent miss)
    if (DYN && seeds && k >= 0) (void)P.at(rc ? (int64_t)len - 1 - k : k);
  };
  uint32_t pend = 0, csym = 0;                           // STEP 3: hi's rank deferred to the next iteration
  auto step = [&]() {                                    // one backward step (LF mapping)
    if (STEP == 3) {
      // k stays put while hi's rank is pending, so the symbol is simply re-read (no divergence)
      csym = rc ? 3u - P.at((int64_t)len - 1 - k) : P.at(k);
      uint32_t nl;
      const bool done = BW == 1 ? fm_step_pend_x2<SMS>(F, C4, csym, lo, hi, pend, nl)
                                : fm_step_pend<SMS>(F, C4, csym, lo, hi, pend, nl);
      if (done) --k;
      if (WORK) { n_steps += pend ? 0 : 1; n_lines += nl; }
      return;
    }
    const uint32_t c = rc ? 3u - P.at((int64_t)len - 1 - k) : P.at(k);
    uint32_t nl;
    if (BW == 1)        fm_step_x2<SMS>(F, c, lo, hi, nl, &C4);
    else if (STEP == 2) fm_step_lean<SMS>(F, C4, c, lo, hi, nl);
    else if (STEP == 4) fm_step_cont<0>(F, c, lo, hi, nl);
    else                fm_step<SMS, 0>(F, c, lo, hi, nl);
    --k;
    if (WORK) { n_steps += 1; n_lines += nl; }
  };
  auto finish = [&]() {
    const uint32_t cnt = lo < hi ? hi - lo : 0u;
    if (STRANDS == 2 && rc) out_rc[ti >> 1] = cnt;
    else out[STRANDS == 2 ? ti >> 1 : ti] = cnt;
  };
  if (!DYN) {
    if (ti < ntask) seed();
    while (ti < ntask) {
      if (pend || (k >= 0 && lo < hi)) step();
      if (!pend && (k < 0 || lo >= hi)) {                // finished: write, claim the next task
        finish();
        ti += stride;
        if (ti < ntask) seed();
      }
    }
  } else {
    const uint32_t lane = threadIdx.x & 31u;
    uint64_t cb = 0, ce = 0;                             // the warp's chunk [cb, ce) (warp-uniform)
    bool exhausted = false, has = false;
    while (true) {
      if (has) {
        if (pend || (k >= 0 && lo < hi)) step();
        if (!pend && (k < 0 || lo >= hi)) { finish(); has = false; }
      }
      const uint32_t needm = __ballot_sync(0xffffffffu, !has);
      if (needm && !exhausted) {
        const uint32_t cnt = __popc(needm), r = __popc(needm & ((1u << lane) - 1u));
        const uint64_t avail = ce - cb;
        uint64_t nb = 0, ne = 0;
        if (cnt > avail) {                               // top up from a fresh chunk
          if (lane == 0) nb = atomicAdd(ctr, (unsigned long long)FM_CHUNK);
          nb = __shfl_sync(0xffffffffu, nb, 0);
          ne = nb + FM_CHUNK < ntask ? nb + FM_CHUNK : ntask;
          if (nb >= ntask) { exhausted = true; nb = ne = ntask; }
        }
        if (!has) {
          const uint64_t t = r < avail ? cb + r : nb + (r - avail);
          if (r < avail || t < ne) { ti = t; seed(); has = true; }
        }
        if (cnt > avail) {
          const uint64_t take = cnt - avail;
          cb = nb + take < ne ? nb + take : ne;
          ce = ne;
        } else {
          cb += cnt;
        }
      }
      if (exhausted && __ballot_sync(0xffffffffu, has) == 0) break;
    }
  }
  if (WORK && n_steps) {
    atomicAdd(work, (unsigned long long)n_steps);
    atomicAdd(work + 1, (unsigned long long)n_lines);
  }
}

// ---- count kernel for L2-resident BWTs (default there; knob fm_step = 3 forces it) ---------
// Instruction-bound regime (configs[3]: the 18-21 MB BWT sits in L2, ncu issue-active ~70-75%),
// so every issue slot counts:
//  * one line per loop iteration (fm_step_pend / fm_step_pend_x2): lo and hi of a step share the
//    line, its delta, superblock word and C[c] whenever they share a half line;
//  * the step runs unconditionally in every lane — lanes without a live task compute on their
//    last (valid) interval and discard the result — so no lane of a warp diverges around it
//    (ncu of the guarded loop: its body ran 1.32x per iteration because lanes entering with a
//    pending rank took a separate path);
//  * lanes are refilled from the warp's task chunk only once at least `refill_min` of them are
//    idle: the refill (seed load, pattern pointer) ran in ~93% of iterations with ~3 of 32 lanes
//    active, ~80 issue slots each time;
//  * seeds come from the k_fm_seed pre-pass (one 8-byte load per task).
// 5 resident CTAs (47 / 44 registers, no spills): configs[3] 9.48 -> 9.58 G patterns/s; 6 spills
#ifndef QR_FM_L2_MINB
#define QR_FM_L2_MINB 5
#endif
template <bool FIXED, bool WORK, int STRANDS, int SMS, int BW, bool PACKED>
__global__ void __launch_bounds__(256, QR_FM_L2_MINB) k_fm_count_l2(FmParams F, const uint8_t* __restrict__ pat,
                                                              const uint64_t* __restrict__ offs,
                                                              const uint32_t* __restrict__ lens, uint32_t fixed_len,
                                                              uint32_t* __restrict__ out, uint32_t* __restrict__ out_rc,
                                                              uint64_t m, unsigned long long* __restrict__ work,
                                                              unsigned long long* __restrict__ ctr,
                                                              const void* __restrict__ seeds_, uint32_t refill_min) {
  if (BW == 1) x2_masks_init();
  fm_preload_super<SMS>(F);
  const uint64_t ntask = m * STRANDS;
  const uint4 C4 = __ldg(reinterpret_cast<const uint4*>(F.Ct));
  const uint32_t lane = threadIdx.x & 31u;
  uint64_t ti = 0;
  uint32_t lo = 0, hi = 0, len = 0, rc = 0, pend = 0;
  // packed seeds: patterns of <= 46 symbols, so the step counter fits 32 bits (no 64-bit compares)
  typename std::conditional<PACKED, int32_t, int64_t>::type k = -1;
  bool has = false;
  PatWindow P;
  P.reset(pat);
  uint64_t sy = 0;                                       // PACKED: the remaining symbols, next in bits 0-1
  uint64_t n_steps = 0, n_lines = 0;
  uint64_t cb = 0, ce = 0;                               // the warp's chunk [cb, ce) (warp-uniform)
  bool exhausted = false;
  while (true) {
    const uint32_t needm = __ballot_sync(0xffffffffu, !has);
    const uint32_t cnt = __popc(needm);
    if (cnt && !exhausted && (cnt >= refill_min || cnt == 32u)) {
      const uint32_t r = __popc(needm & ((1u << lane) - 1u));
      const uint64_t avail = ce - cb;
      uint64_t nb = 0, ne = 0;
      if (cnt > avail) {                                 // top up from a fresh chunk
        if (lane == 0) nb = atomicAdd(ctr, (unsigned long long)FM_CHUNK);
        nb = __shfl_sync(0xffffffffu, nb, 0);
        ne = nb + FM_CHUNK < ntask ? nb + FM_CHUNK : ntask;
        if (nb >= ntask) { exhausted = true; nb = ne = ntask; }
      }
      if (!has) {
        const uint64_t t = r < avail ? cb + r : nb + (r - avail);
        if (r < avail || t < ne) {
          ti = t;
          const uint64_t pi = STRANDS == 2 ? ti >> 1 : ti;
          rc = STRANDS == 2 ? (uint32_t)(ti & 1) : 0u;
          len = FIXED ? fixed_len : lens[pi];
          if (PACKED) {
            const uint4 sv = __ldg(reinterpret_cast<const uint4*>(seeds_) + ti);
            lo = sv.x;
            hi = sv.y;
            sy = ((uint64_t)sv.w << 32) | sv.z;
          } else {
            P.reset(pat + (FIXED ? pi * (uint64_t)fixed_len : offs[pi]));
            const uint2 iv = __ldg(reinterpret_cast<const uint2*>(seeds_) + ti);
            lo = iv.x;
            hi = iv.y;
          }
          k = (decltype(k))len - 1 - ((F.K && len >= (uint32_t)F.K) ? F.K : 0);
          pend = 0;
          has = true;
        }
      }
      if (cnt > avail) {
        const uint64_t take = cnt - avail;
        cb = nb + take < ne ? nb + take : ne;
        ce = ne;
      } else {
        cb += cnt;
      }
    }
    if (exhausted && __ballot_sync(0xffffffffu, has) == 0) break;
    // one line of one backward step, in every lane (results kept only where act)
    const bool act = has && (pend || (k >= 0 && lo < hi));
    uint32_t c;
    if (PACKED) {
      c = (uint32_t)sy & 3u;
    } else {
      const int64_t idx = rc ? (int64_t)len - 1 - k : k;
      c = P.at_if(act, idx) ^ (rc ? 3u : 0u);
    }
    uint32_t nlo = lo, nhi = hi, npend = pend, nl;
    const bool done = BW == 1 ? fm_step_pend_x2<SMS>(F, C4, c, nlo, nhi, npend, nl)
                              : fm_step_pend<SMS>(F, C4, c, nlo, nhi, npend, nl);
    if (WORK && act) { n_steps += pend ? 0u : 1u; n_lines += nl; }
    lo = act ? nlo : lo;
    hi = act ? nhi : hi;
    pend = act ? npend : pend;
    k -= (act && done) ? 1 : 0;
    if (PACKED) sy = (act && done) ? sy >> 2 : sy;
    if (has && !pend && (k < 0 || lo >= hi)) {           // finished: write the count
      const uint32_t res = lo < hi ? hi - lo : 0u;
      if (STRANDS == 2 && rc) out_rc[ti >> 1] = res;
      else out[STRANDS == 2 ? ti >> 1 : ti] = res;
      has = false;
    }
  }
  if (WORK && n_steps) {
    atomicAdd(work, (unsigned long long)n_steps);
    atomicAdd(work + 1, (unsigned long long)n_lines);
  }
}

// ---- approximate counting with <= 1 substitution (NEXT §8(f)3) ---------------------------
// The paper motivates rank_4 by approximate matching in an FM index: one
// rank_4 at lo and one at hi give the four extensions of an interval at once.  A text position
// matches P with at most one substitution in exactly one way (exactly, or with the single
// mismatch at a unique position j and text symbol c), so
//   count_{<=1}(P) = |exact interval| + sum_j sum_{c != P[j]} |backward search of P[0..j) from
//                    extend(I_{j+1}, c)|,
// where I_{j+1} is the exact interval of P[j+1..).  Mismatches inside the pattern's last 8
// symbols read their extended interval straight from the 8-mer table (24 substituted keys);
// the others branch from the exact path with rank_4.  Each branch continues as an exact
// backward search and usually dies within a few steps.

// rank_4 over a QuadRank16x2 BWT at row x (one sector; plane popcounts as q16x2_rank4).
__device__ __forceinline__ void fm_occ4_x2(const FmParams& F, uint32_t x, uint32_t occ[4]) {
  uint32_t j, h, p;
  x2_locate(x, (uint32_t)F.last_line, j, h, p);
  uint64_t w[4];
  ld_sector(F.lines + 4 * (uint64_t)j + 2 * h, w[0], w[1], w[2], w[3]);
  const uint4 sv = __ldg(reinterpret_cast<const uint4*>(F.super) + (j >> QD_SB_LOG));
  const uint4 mm = reinterpret_cast<const uint4*>(g_x2_masks)[p];
  const uint64_t m0 = ((uint64_t)mm.y << 32) | mm.x, m1 = ((uint64_t)mm.w << 32) | mm.z;
  const uint64_t l0 = w[1] & m0, h0 = w[2] & m0, l1 = w[3] & m1, h1 = (w[3] >> 32) & m1;
  const uint32_t nl = __popcll(l0) + __popcll(l1), nh = __popcll(h0) + __popcll(h1);
  const uint32_t nt = __popcll(l0 & h0) + __popcll(l1 & h1);
  const uint32_t len = p >= 48 ? p - 48u : 48u - p;
  const uint32_t cnt[4] = {len - nl - nh + nt, nl - nt, nh - nt, nt};
  const uint32_t s4[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t base = (s4[c] << QD_SHIFT) + (uint32_t)((w[0] >> (16 * c)) & 0xffffull);
    occ[c] = p >= 48 ? base + cnt[c] : base - cnt[c];
  }
  occ[0] -= (x > (uint32_t)F.spos);
}

// rank_4 over the BWT at row x (Occ of all four symbols, '$' correction on A).
__device__ __forceinline__ void fm_occ4(const FmParams& F, uint32_t x, uint32_t occ[4]) {
  uint32_t j = (x >> 5) / 7u;
  j = j > (uint32_t)F.last_line ? (uint32_t)F.last_line : j;
  const uint32_t p = 32u + x - j * (uint32_t)QD_B;
  const uint4* L = F.lines + 4 * (uint64_t)j;
  const bool right = p >= 128;
  // the counted half's sector, and (right of the anchor) the 16 B of sector 0 holding the deltas:
  // 6 live u64 instead of both sectors' 8 (the backtracking kernels are register-bound)
  uint64_t w[4];
  ld_sector(L + (right ? 2 : 0), w[0], w[1], w[2], w[3]);
  uint64_t a[2];
  if (right) {
    const ulonglong2 dv = __ldg(reinterpret_cast<const ulonglong2*>(L));
    a[0] = dv.x; a[1] = dv.y;
  } else {
    a[0] = w[0]; a[1] = w[1];
  }
  const uint4 sv = __ldg(reinterpret_cast<const uint4*>(F.super) + (j >> QD_SB_LOG));
  const int xx = (int)(p & 127u);
  const uint64_t inv = right ? 0ull : ~0ull;
  uint32_t nl = 0, nh = 0, nt = 0;
  uint64_t mk[2];
  qd_masks((uint32_t)xx, mk[0], mk[1]);
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    uint64_t msk = mk[t] ^ inv;
    uint64_t l = ~w[2 * t] & msk, hh = ~w[2 * t + 1] & msk;
    nl += __popcll(l);
    nh += __popcll(hh);
    nt += __popcll(l & hh);
  }
  const uint32_t len = right ? (uint32_t)xx : 128u - (uint32_t)xx;
  const uint32_t cnt[4] = {len - nl - nh + nt, nl - nt, nh - nt, nt};
  const uint32_t s4[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint64_t dw = (c & 2) ? a[1] : a[0];
    const uint32_t base = (s4[c] << QD_SHIFT) + (uint32_t)((dw >> (16 * (c & 1))) & 0xffffull);
    occ[c] = right ? base + cnt[c] : base - cnt[c];
  }
  occ[0] -= (x > (uint32_t)F.spos);
}

// exact backward search of P[0..k] from [lo, hi); returns the final interval size
// the same for three intervals continuing over the same symbols P[k], P[k-1], ...: their steps
// are independent, so each position issues the loads of all live intervals before consuming any
// Work accounting of the approximate-search kernels (WORK = true, qr_fm_count_work_ex): ws counts
// rank evaluations at an interval's two ends (exact steps, rank_4 pairs) plus k-mer table
// lookups, wl the distinct lines (table entries) they gather.
struct FmWork {
  uint64_t ws = 0, wl = 0;
};
template <int BW>
__device__ __forceinline__ uint32_t fm_line_of(const FmParams& F, uint32_t x) {
  uint32_t j = BW == 1 ? (x >> 6) / 3u : (x >> 5) / 7u;
  return j > (uint32_t)F.last_line ? (uint32_t)F.last_line : j;
}

#ifndef QR_CONT3_COMPACT
#define QR_CONT3_COMPACT 1
#endif
template <int BW, bool WORK = false, class W>
__device__ __forceinline__ uint32_t fm_continue3(const FmParams& F, W& P, int64_t k, uint32_t (&lo)[3],
                                                 uint32_t (&hi)[3], FmWork& wk) {
  uint32_t nl;
#if QR_CONT3_COMPACT
  // The live intervals are kept first (compacted after every step), so the step of slot 0 runs
  // for every lane still in the loop and slots 1, 2 only for lanes with 2, 3 live intervals:
  // unordered, each of the three step copies ran with the subset of lanes whose interval r was
  // live (~3 of 32 lanes per instruction on the 150-bp reads, ncu).
  auto compact = [&]() {
    if (!(lo[1] < hi[1])) { lo[1] = lo[2]; hi[1] = hi[2]; lo[2] = hi[2] = 0u; }
    if (!(lo[0] < hi[0])) { lo[0] = lo[1]; hi[0] = hi[1]; lo[1] = lo[2]; hi[1] = hi[2]; lo[2] = hi[2] = 0u; }
  };
  compact();
  for (; k >= 0 && lo[0] < hi[0]; --k) {
    const uint32_t c = P.at(k);
    fm_step_cont<BW>(F, c, lo[0], hi[0], nl);
    if (WORK) { wk.ws += 1; wk.wl += nl; }
#pragma unroll
    for (int r = 1; r < 3; ++r)
      if (lo[r] < hi[r]) {
        fm_step_cont<BW>(F, c, lo[r], hi[r], nl);
        if (WORK) { wk.ws += 1; wk.wl += nl; }
      }
    compact();
  }
#else
  for (; k >= 0 && (lo[0] < hi[0] || lo[1] < hi[1] || lo[2] < hi[2]); --k) {
    const uint32_t c = P.at(k);
#pragma unroll
    for (int r = 0; r < 3; ++r)
      if (lo[r] < hi[r]) {
        fm_step_cont<BW>(F, c, lo[r], hi[r], nl);
        if (WORK) { wk.ws += 1; wk.wl += nl; }
      }
  }
#endif
  uint32_t t = 0;
#pragma unroll
  for (int r = 0; r < 3; ++r) t += lo[r] < hi[r] ? hi[r] - lo[r] : 0u;
  return t;
}

template <int BW, bool WORK = false, class W>
__device__ __forceinline__ uint32_t fm_continue(const FmParams& F, W& P, int64_t k, uint32_t lo, uint32_t hi,
                                                FmWork& wk) {
  uint32_t nl;
  for (; k >= 0 && lo < hi; --k) {
    fm_step_cont<BW>(F, P.at(k), lo, hi, nl);
    if (WORK) { wk.ws += 1; wk.wl += nl; }
  }
  return lo < hi ? hi - lo : 0u;
}
// rank_4 at both ends of an interval (the four children of a search-tree node)
template <int BW, bool WORK>
__device__ __forceinline__ void fm_occ4_pair(const FmParams& F, uint32_t lo, uint32_t hi, uint32_t (&ol)[4],
                                             uint32_t (&oh)[4], FmWork& wk) {
  if (BW == 1) { fm_occ4_x2(F, lo, ol); fm_occ4_x2(F, hi, oh); }
  else         { fm_occ4(F, lo, ol); fm_occ4(F, hi, oh); }
  if (WORK) { wk.ws += 1; wk.wl += fm_line_of<BW>(F, lo) == fm_line_of<BW>(F, hi) ? 1u : 2u; }
}

// Table entry of the approximate search.  Over a text with fewer distinct K-mers than 4^K / 2
// most of the substituted K-mers a search looks up are absent (configs[3], n = 2^26, K = 14: 78%);
// a presence bitmap of the table (4^K bits: 32 MiB at K = 14, L2-resident next to the BWT)
// answers those from the L2 instead of reading the 2-GiB table from HBM.
__device__ __forceinline__ uint2 ax_lookup(const FmParams& F, uint32_t key) {
  if (F.kbits && !((__ldg(F.kbits + (key >> 5)) >> (key & 31u)) & 1u)) return make_uint2(0u, 0u);
  return ld_kmer(F.kmer + key);
}

// key with the symbol at key position t replaced by (old + r) mod 4, r in 1..3
__device__ __forceinline__ uint32_t kmer_subst(uint32_t key, int t, uint32_t r) {
  const uint32_t o = (key >> (2 * t)) & 3u;
  return key ^ ((o ^ ((o + r) & 3u)) << (2 * t));
}

// Presence of the three substitutions at key position t (bit r - 1: symbol (old + r) mod 4).
__device__ __forceinline__ uint32_t ax_present3(const FmParams& F, uint32_t key, int t) {
  uint32_t m = 0;
#pragma unroll
  for (uint32_t r = 1; r < 4; ++r) {
    const uint32_t k = kmer_subst(key, t, r);
    m |= ((__ldg(F.kbits + (k >> 5)) >> (k & 31u)) & 1u) << (r - 1);
  }
  return m;
}

// The last substitution level of a seeded search: every K-mer one substitution away from key at
// a position t in [t0, K) (3 (K - t0) variants) is looked up and continued as an exact search
// from pattern position pos - 1, the three variants of a position together (fm_continue3).  With
// the presence bitmap all 3 (K - t0) probes are issued first (independent L2 loads) and only the
// positions with a present variant are looked up and continued.
template <int BW, bool WORK, class W>
__device__ __forceinline__ uint64_t ax_last_levels(const FmParams& F, W& P, uint32_t key, int t0, uint32_t pos,
                                                   FmWork& wk) {
  const int nb = 3 * (F.K - t0);                          // <= 42 (K <= 14)
  uint64_t pm = nb > 0 ? ~0ull >> (64 - nb) : 0ull;
  if (F.kbits) {
    pm = 0;
    for (int t = t0; t < F.K; ++t) pm |= (uint64_t)ax_present3(F, key, t) << (3 * (t - t0));
  }
  if (WORK && nb > 0) { wk.ws += (uint32_t)nb; wk.wl += (uint32_t)nb; }   // one table lookup per variant
  uint64_t total = 0;
  while (pm) {
    const int sh = 3 * ((__ffsll((long long)pm) - 1) / 3);
    const uint32_t g = (uint32_t)(pm >> sh) & 7u;
    pm &= ~(7ull << sh);
    const int t = t0 + sh / 3;
    uint2 iv[3];
#pragma unroll
    for (uint32_t r = 1; r < 4; ++r)
      iv[r - 1] = (g >> (r - 1)) & 1u ? ld_kmer(F.kmer + kmer_subst(key, t, r)) : make_uint2(0u, 0u);
    uint32_t vl[3] = {iv[0].x, iv[1].x, iv[2].x}, vh[3] = {iv[0].y, iv[1].y, iv[2].y};
    total += fm_continue3<BW, WORK>(F, P, (int64_t)pos - 1, vl, vh, wk);
  }
  return total;
}

// bits[w] bit i = (table[32 w + i] is non-empty); every lane of a warp runs the same iterations
__global__ void k_kmer_bits(const uint2* __restrict__ table, uint64_t entries, uint32_t* __restrict__ bits) {
  const uint64_t ent32 = (entries + 31) & ~31ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ent32; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 v = i < entries ? table[i] : make_uint2(0u, 0u);
    const uint32_t b = __ballot_sync(0xffffffffu, v.x < v.y);
    if ((threadIdx.x & 31u) == 0) bits[i >> 5] = b;
  }
}

// Next pattern index of a lane.  Static: grid stride.  Dynamic (ctr != null): the lanes that reach
// this point together (__activemask) take consecutive indices with one atomicAdd by the first of
// them, so a lane that finishes its pattern starts another at once instead of idling until the
// slowest pattern of the static assignment (the work per pattern varies by branch count).
__device__ __forceinline__ uint64_t approx_next(unsigned long long* ctr, uint64_t cur, uint64_t stride) {
  if (!ctr) return cur + stride;
  const uint32_t am = __activemask();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t leader = __ffs(am) - 1u;
  unsigned long long b = 0;
  if (lane == leader) b = atomicAdd(ctr, (unsigned long long)__popc(am));
  b = __shfl_sync(am, b, leader);
  return b + __popc(am & ((1u << lane) - 1u));
}

// k = 2 (k_fm_approxk) runs 4 CTAs per SM too (64 registers, ~100 B of spills): since the frames
// moved to shared memory, the extra warps beat the spills — +4.5% (BWT16) / +5% (150-bp reads),
// BWT16x2 unchanged (profiles/r02_approx_minb.log; round 1's register-resident frames measured
// -3% with the same bound).  k = 3 runs 3 (80 registers): since the presence bitmap batches its
// last-level probes, +10% over 4 CTAs on BWT16, +1% on BWT16x2 (profiles/r02_approx_kbits.log).
#ifndef QR_APPROX_MINB
#define QR_APPROX_MINB 4
#endif
#ifndef QR_APPROX3_MINB
#define QR_APPROX3_MINB 3
#endif
#define QR_APPROX_LB __launch_bounds__(256, KMAX == 3 ? QR_APPROX3_MINB : QR_APPROX_MINB)
// k = 1 runs 4 CTAs per SM (64 registers): +10% on the HBM-resident 150-bp reads, where the
// search waits on DRAM (profiles/r01_reads_approx_minblocks.jsonl)
#ifndef QR_APPROX1_MINB
#define QR_APPROX1_MINB 4
#endif

template <bool FIXED, int BW, int STRANDS, bool WORK = false>
__global__ void __launch_bounds__(256, QR_APPROX1_MINB) k_fm_approx1(FmParams F, const uint8_t* __restrict__ pat,
                                                    const uint64_t* __restrict__ offs,
                                                    const uint32_t* __restrict__ lens, uint32_t fixed_len,
                                                    uint32_t* __restrict__ out, uint32_t* __restrict__ out_rc,
                                                    uint64_t m, unsigned long long* __restrict__ ctr,
                                                    unsigned long long* __restrict__ work) {
  FmWork wk;
  if (BW == 1) x2_masks_init();
  else qd_masks_init();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint4 C4 = __ldg(reinterpret_cast<const uint4*>(F.Ct));
  const uint32_t Cs[4] = {C4.x, C4.y, C4.z, C4.w};
  const uint64_t ntask = m * STRANDS;
  for (uint64_t ti = ctr ? approx_next(ctr, 0, 0) : blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ti < ntask;
       ti = approx_next(ctr, ti, stride)) {
    const uint64_t pi = STRANDS == 2 ? ti >> 1 : ti;
    const uint32_t rc = STRANDS == 2 ? (uint32_t)(ti & 1) : 0u;
    const uint32_t len = FIXED ? fixed_len : lens[pi];
    const uint8_t* p = pat + (FIXED ? pi * (uint64_t)fixed_len : offs[pi]);
    StrandWindow<STRANDS> P;
    P.reset(p, len, rc);
    uint64_t total = 0;
    uint32_t lo, hi;
    int64_t j;
    if (F.K && len >= (uint32_t)F.K) {
      const uint32_t key0 = rc ? kmer_key_rc(F.K, P.P, p, len) : kmer_key(F.K, P.P, p, len);
      // one substitution among the last K symbols
      total += ax_last_levels<BW, WORK>(F, P, key0, 0, len - (uint32_t)F.K, wk);
      const uint2 iv0 = ax_lookup(F, key0);
      if (WORK) { wk.ws += 1; wk.wl += 1; }
      lo = iv0.x; hi = iv0.y;
      j = (int64_t)len - 1 - F.K;
    } else {
      lo = 0; hi = (uint32_t)F.N;
      j = (int64_t)len - 1;
    }
    for (; j >= 0 && lo < hi; --j) {                     // exact path; branch on the mismatch at j
      uint32_t ol[4], oh[4];
      fm_occ4_pair<BW, WORK>(F, lo, hi, ol, oh, wk);
      const uint32_t cj = P.at(j);
      uint32_t bl[3], bh[3];                              // the three substituted symbols' intervals
#pragma unroll
      for (uint32_t r = 0; r < 3; ++r) {
        const uint32_t c = (cj + 1 + r) & 3u;
        bl[r] = Cs[c] + ol[c];
        bh[r] = Cs[c] + oh[c];
      }
      total += fm_continue3<BW, WORK>(F, P, j - 1, bl, bh, wk);
      lo = Cs[cj] + ol[cj];
      hi = Cs[cj] + oh[cj];
    }
    if (lo < hi) total += hi - lo;
    if (STRANDS == 2 && rc) out_rc[pi] = (uint32_t)total;
    else out[pi] = (uint32_t)total;
  }
  if (WORK && wk.ws) {
    atomicAdd(work, (unsigned long long)wk.ws);
    atomicAdd(work + 1, (unsigned long long)wk.wl);
  }
}

// ---- approximate counting with <= KMAX substitutions, KMAX = 2, 3 ---------------------------
// Backtracking over the BWT with rank_4 at every node: a node is an interval
// [lo, hi) after the pattern's last symbols with mm substitutions so far; one rank_4 at lo and
// one at hi give all four children, the child on the pattern's symbol keeps mm and the other
// three (when mm < KMAX) are new nodes with mm + 1.  The search keeps one frame per mismatch
// level: frame f walks the exact path of its node and, at each position, first descends into
// the mismatched children (frame f + 1) before stepping on, so the state is KMAX + 1 frames
// whatever the pattern length.  Frames at mm = KMAX finish as plain exact searches.  Leaves are
// distinct strings, so their interval sizes add up to the number of text positions within
// Hamming distance KMAX.
//
// Seeding: the first K levels of the tree (the pattern's last K symbols) are not expanded node
// by node; every K-mer within distance KMAX of the pattern's last K symbols is looked up in the
// k-mer table instead (1 + 3K + 9 C(K,2) [+ 27 C(K,3)] lookups), and the search continues from
// each non-empty interval with the substitutions it has left.
// The search frames live in shared memory, word-major with a stride of the CTA size (256), so a
// warp's accesses to one field are 32 consecutive words (no bank conflict): indexed by the frame
// number at run time they would otherwise sit in the local-memory stack (112 B per thread at
// k = 2) and compete with the BWT gathers for the L1, and hold ~14 registers.
template <int KMAX>
struct FmFrames {
  static constexpr int WORDS = 4 * (KMAX + 1) + 8 * KMAX;   // lo, hi, pos, next branch per frame; children
  uint32_t* b;
  __device__ __forceinline__ explicit FmFrames(uint32_t* smem) : b(smem + threadIdx.x) {}
  __device__ __forceinline__ uint32_t& lo(int f) { return b[(0 * (KMAX + 1) + f) * 256]; }
  __device__ __forceinline__ uint32_t& hi(int f) { return b[(1 * (KMAX + 1) + f) * 256]; }
  __device__ __forceinline__ uint32_t& pos(int f) { return b[(2 * (KMAX + 1) + f) * 256]; }
  __device__ __forceinline__ uint32_t& nd(int f) { return b[(3 * (KMAX + 1) + f) * 256]; }
  __device__ __forceinline__ uint32_t& clo(int f, int c) { return b[(4 * (KMAX + 1) + 4 * f + c) * 256]; }
  __device__ __forceinline__ uint32_t& chi(int f, int c) { return b[(4 * (KMAX + 1) + 4 * KMAX + 4 * f + c) * 256]; }
};

template <int BW, int KMAX, bool WORK, class W>
__device__ __forceinline__ uint64_t fm_backtrack(const FmParams& F, W& P, const uint32_t (&Cs)[4],
                                                 uint32_t lo, uint32_t hi, uint32_t pos, int f0, FmWork& wk,
                                                 FmFrames<KMAX>& fr) {
  constexpr uint32_t UNX = 8;   // not 4: a frame whose branches are all tried has nd = 4
  uint64_t total = 0;
  int f = f0;
  fr.lo(f) = lo; fr.hi(f) = hi; fr.pos(f) = pos; fr.nd(f) = UNX;
  while (f >= f0) {
    const uint32_t flo = fr.lo(f), fhi = fr.hi(f), fpos = fr.pos(f);
    uint32_t d = fr.nd(f);
    if (d == UNX) {
      if (flo >= fhi) { --f; continue; }
      if (fpos == 0) { total += fhi - flo; --f; continue; }
      if (f == KMAX) {                                   // no substitution left: exact search
        total += fm_continue<BW, WORK>(F, P, (int64_t)fpos - 1, flo, fhi, wk);
        --f;
        continue;
      }
      uint32_t ol[4], oh[4];
      fm_occ4_pair<BW, WORK>(F, flo, fhi, ol, oh, wk);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        fr.clo(f, c) = Cs[c] + ol[c];
        fr.chi(f, c) = Cs[c] + oh[c];
      }
      d = 0;
    }
    const uint32_t pc = P.at((int64_t)fpos - 1);
    while (d < 4 && (d == pc || fr.clo(f, d) >= fr.chi(f, d))) ++d;
    if (d < 4) {                                         // descend into the substitution d
      fr.nd(f) = d + 1;
      fr.lo(f + 1) = fr.clo(f, d); fr.hi(f + 1) = fr.chi(f, d); fr.pos(f + 1) = fpos - 1; fr.nd(f + 1) = UNX;
      ++f;
      continue;
    }
    fr.lo(f) = fr.clo(f, pc); fr.hi(f) = fr.chi(f, pc); fr.pos(f) = fpos - 1; fr.nd(f) = UNX;   // step on the pattern's symbol
  }
  return total;
}


template <bool FIXED, int BW, int KMAX, int STRANDS, bool WORK = false>
__global__ void QR_APPROX_LB k_fm_approxk(FmParams F, const uint8_t* __restrict__ pat,
                                                    const uint64_t* __restrict__ offs,
                                                    const uint32_t* __restrict__ lens, uint32_t fixed_len,
                                                    uint32_t* __restrict__ out, uint32_t* __restrict__ out_rc,
                                                    uint64_t m, unsigned long long* __restrict__ ctr,
                                                    unsigned long long* __restrict__ work) {
  FmWork wk;
  if (BW == 1) x2_masks_init();
  else qd_masks_init();
  extern __shared__ uint32_t fm_frames_smem[];
  FmFrames<KMAX> fr(fm_frames_smem);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint4 C4 = __ldg(reinterpret_cast<const uint4*>(F.Ct));
  const uint32_t Cs[4] = {C4.x, C4.y, C4.z, C4.w};
  const uint64_t ntask = m * STRANDS;
  for (uint64_t ti = ctr ? approx_next(ctr, 0, 0) : blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ti < ntask;
       ti = approx_next(ctr, ti, stride)) {
    const uint64_t pi = STRANDS == 2 ? ti >> 1 : ti;
    const uint32_t rc = STRANDS == 2 ? (uint32_t)(ti & 1) : 0u;
    const uint32_t len = FIXED ? fixed_len : lens[pi];
    const uint8_t* p = pat + (FIXED ? pi * (uint64_t)fixed_len : offs[pi]);
    StrandWindow<STRANDS> P;
    P.reset(p, len, rc);
    uint64_t total = 0;
    const int K = F.K;
    if (K && len >= (uint32_t)K) {
      const uint32_t key0 = rc ? kmer_key_rc(K, P.P, p, len) : kmer_key(K, P.P, p, len);
      const uint32_t pos = len - (uint32_t)K;
      auto seed = [&](uint32_t key, int mm) {
        const uint2 iv = ax_lookup(F, key);
        if (WORK) { wk.ws += 1; wk.wl += 1; }
        if (iv.x < iv.y) total += fm_backtrack<BW, KMAX, WORK>(F, P, Cs, iv.x, iv.y, pos, mm, wk, fr);
      };
      // the seeds with all KMAX substitutions inside the K-mer have none left: the variants at the
      // last substituted position are looked up and continue as exact searches (ax_last_levels)
      seed(key0, 0);
      for (int t1 = 0; t1 < K; ++t1)
        for (uint32_t r1 = 1; r1 < 4; ++r1) {
          const uint32_t k1 = kmer_subst(key0, t1, r1);
          seed(k1, 1);
          if (KMAX == 2) {
            total += ax_last_levels<BW, WORK>(F, P, k1, t1 + 1, pos, wk);
          } else {
            for (int t2 = t1 + 1; t2 < K; ++t2)
              for (uint32_t r2 = 1; r2 < 4; ++r2) {
                const uint32_t k2 = kmer_subst(k1, t2, r2);
                seed(k2, 2);
                total += ax_last_levels<BW, WORK>(F, P, k2, t2 + 1, pos, wk);
              }
          }
        }
    } else {
      total = fm_backtrack<BW, KMAX, WORK>(F, P, Cs, 0u, (uint32_t)F.N, len, 0, wk, fr);
    }
    if (STRANDS == 2 && rc) out_rc[pi] = (uint32_t)total;
    else out[pi] = (uint32_t)total;
  }
  if (WORK && wk.ws) {
    atomicAdd(work, (unsigned long long)wk.ws);
    atomicAdd(work + 1, (unsigned long long)wk.wl);
  }
}

// ---- approximate counting with <= k substitutions (k = 1, 2), breadth first ------------------
// The same decomposition as the recursive kernels (a leaf of the substitution tree is a distinct
// string; PAPER.md:139-140 — rank_4 at both ends of a node gives its four children), run level
// by level (mm = substitutions left) so that every lane of a warp does the same kind of work:
//   k_ax_seed   one thread per task: the exact seed interval of the last K symbols, and the
//               K-mers within distance k of them that the table holds (presence bitmap, or all),
//               written as lookup items (task, key) to one queue per level (exact sizes);
//   k_ax_path   items with mm >= 1: their exact path with rank_4 at both ends (one step per lane
//               and iteration, lanes refilled from the item range); the three substituted
//               children of every step go to the queue of level mm - 1 as interval items
//               (task, pos, lo, hi);
//   k_ax_cont   items with mm = 0: plain exact searches, one step per lane and iteration.
// Each item adds its count to its task's output (the level-k path, one item per task, first).
// In the recursive kernels a lane walks its pattern's tree — the exact path and, at every step,
// the continuations of its branches — so the lanes of a warp sit in different loops (ncu: ~11
// of 32 lanes per instruction) and each lane's dependent gathers serialise behind the others'.
// Interval items that do not fit their queue (sized for ~4 per task) are searched by the
// emitting lane itself (exact continuation, or the recursive one-substitution walk).
__device__ __forceinline__ uint32_t sel4(const uint32_t (&a)[4], uint32_t c) {
  return (c & 2u) ? ((c & 1u) ? a[3] : a[2]) : ((c & 1u) ? a[1] : a[0]);
}
struct AxCtl {                  // device counters of one chunk (zeroed before the chunk)
  unsigned long long z[3];      // lookup-queue sizes by level (mm = substitutions left)
  unsigned long long q[3];      // interval-queue sizes by level
  unsigned long long ctr[10];   // work-order counters of the chunk's launches
};

template <bool FIXED, int STRANDS>
__device__ __forceinline__ const uint8_t* ax_pattern(const uint8_t* pat, const uint64_t* offs, const uint32_t* lens,
                                                     uint32_t fixed_len, uint64_t ti, uint32_t& len, uint32_t& rc) {
  const uint64_t pi = STRANDS == 2 ? ti >> 1 : ti;
  rc = STRANDS == 2 ? (uint32_t)(ti & 1) : 0u;
  len = FIXED ? fixed_len : lens[pi];
  return pat + (FIXED ? pi * (uint64_t)fixed_len : offs[pi]);
}
template <int STRANDS>
__device__ __forceinline__ uint32_t* ax_out(uint32_t* out, uint32_t* out_rc, uint64_t ti) {
  return (STRANDS == 2 && (ti & 1)) ? out_rc + (ti >> 1) : out + (STRANDS == 2 ? ti >> 1 : ti);
}
// this lane's first slot of n items in a queue, one atomic per warp (all 32 lanes call it)
__device__ __forceinline__ unsigned long long warp_reserve(unsigned long long* cnt, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += v;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && tot) base = atomicAdd(cnt, (unsigned long long)tot);
  return __shfl_sync(0xffffffffu, base, 31) + (incl - n);
}
// presence of the 3 (K - t0) one-substitution variants of key at positions t0..K-1 (bit 3(t-t0)+r-1)
__device__ __forceinline__ uint64_t ax_present_from(const FmParams& F, uint32_t key, int t0) {
  const int nb = 3 * (F.K - t0);
  if (nb <= 0) return 0ull;
  if (!F.kbits) return ~0ull >> (64 - nb);
  uint64_t pm = 0;
  for (int t = t0; t < F.K; ++t) pm |= (uint64_t)ax_present3(F, key, t) << (3 * (t - t0));
  return pm;
}
__device__ __forceinline__ uint32_t ax_variant(uint32_t key, int t0, int b) {
  return kmer_subst(key, t0 + b / 3, (uint32_t)(b % 3) + 1);
}
// sizes of the listed variants' intervals (a K-mer that is the whole pattern: nothing to continue)
__device__ __forceinline__ uint32_t ax_sizes(const FmParams& F, uint32_t key, int t0, uint64_t pm) {
  uint32_t s = 0;
  for (; pm; pm &= pm - 1) {
    const uint2 iv = ld_kmer(F.kmer + ax_variant(key, t0, __ffsll((long long)pm) - 1));
    s += iv.x < iv.y ? iv.y - iv.x : 0u;
  }
  return s;
}

// The n-substitution variants inside the K-mer go to level KMAX - n (n = 1..KMAX).
template <bool FIXED, int STRANDS, int KMAX, bool WORK>
__global__ void __launch_bounds__(256) k_ax_seed(FmParams F, const uint8_t* __restrict__ pat,
                                                 const uint64_t* __restrict__ offs, const uint32_t* __restrict__ lens,
                                                 uint32_t fixed_len, uint32_t* __restrict__ out,
                                                 uint32_t* __restrict__ out_rc, uint64_t t0, uint64_t t1,
                                                 uint2* __restrict__ seeds, uint2* __restrict__ z0,
                                                 uint2* __restrict__ z1, uint2* __restrict__ z2, AxCtl* ctl,
                                                 unsigned long long* __restrict__ work) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint2* const zq[3] = {z0, z1, z2};
  uint64_t ws = 0;
  for (uint64_t w0 = t0 + (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull); w0 < t1; w0 += warps * 32) {
    const uint64_t ti = w0 + lane;
    const bool valid = ti < t1;
    bool seeded = false, whole = false;
    uint32_t key0 = 0, direct = 0;
    if (valid) {
      uint32_t len, rc;
      const uint8_t* p = ax_pattern<FIXED, STRANDS>(pat, offs, lens, fixed_len, ti, len, rc);
      uint2 iv0 = make_uint2(0u, (uint32_t)F.N);
      if (F.K && len >= (uint32_t)F.K) {
        PatWindow P;
        P.reset(p);
        key0 = rc ? kmer_key_rc(F.K, P, p, len) : kmer_key(F.K, P, p, len);
        iv0 = ax_lookup(F, key0);
        seeded = true;
        whole = len == (uint32_t)F.K;                     // the variants are leaves
        if (WORK) {
          const uint64_t K = (uint64_t)F.K;
          ws += 1 + 3 * K + (KMAX >= 2 ? 9 * K * (K - 1) / 2 : 0) + (KMAX >= 3 ? 27 * K * (K - 1) * (K - 2) / 6 : 0);
        }
      }
      seeds[ti - t0] = iv0;
    }
    // variants at positions t0.. of `key` (one more substitution than key has) to level lvl
    auto emit = [&](uint32_t key, int tfrom, int lvl) {
      uint64_t pm = seeded ? ax_present_from(F, key, tfrom) : 0ull;
      if (whole) { direct += ax_sizes(F, key, tfrom, pm); pm = 0; }
      unsigned long long at = warp_reserve(&ctl->z[lvl], (uint32_t)__popcll(pm));
      for (; pm; pm &= pm - 1) zq[lvl][at++] = make_uint2((uint32_t)ti, ax_variant(key, tfrom, __ffsll((long long)pm) - 1));
    };
    emit(key0, 0, KMAX - 1);                              // one substitution
    if (KMAX >= 2) {
      for (int a1 = 0; a1 < F.K; ++a1)
        for (uint32_t r1 = 1; r1 < 4; ++r1) {
          const uint32_t k1 = kmer_subst(key0, a1, r1);
          emit(k1, a1 + 1, KMAX - 2);                     // two substitutions
          if (KMAX >= 3)
            for (int a2 = a1 + 1; a2 < F.K; ++a2)
              for (uint32_t r2 = 1; r2 < 4; ++r2) emit(kmer_subst(k1, a2, r2), a2 + 1, KMAX - 3);   // three
        }
    }
    if (valid) *ax_out<STRANDS>(out, out_rc, ti) = direct;
  }
  if (WORK && ws) { atomicAdd(work, (unsigned long long)ws); atomicAdd(work + 1, (unsigned long long)ws); }
}

// k = 3: the 9828 (K = 14) variant probes of a task are spread over K threads (task, first
// substituted position a1), so that a chunk of ~18K tasks still fills the GPU; loop bounds are
// warp-uniform (inactive positions emit nothing) so every lane reaches each warp_reserve.
template <int STRANDS>
__global__ void k_ax_zero(uint32_t* __restrict__ out, uint32_t* __restrict__ out_rc, uint64_t t0, uint64_t t1) {
  for (uint64_t ti = t0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; ti < t1; ti += (uint64_t)gridDim.x * blockDim.x)
    *ax_out<STRANDS>(out, out_rc, ti) = 0u;
}
template <bool FIXED, int STRANDS, int KMAX, bool WORK>
__global__ void __launch_bounds__(256) k_ax_seed3(FmParams F, const uint8_t* __restrict__ pat,
                                                  const uint64_t* __restrict__ offs, const uint32_t* __restrict__ lens,
                                                  uint32_t fixed_len, uint32_t* __restrict__ out,
                                                  uint32_t* __restrict__ out_rc, uint64_t t0, uint64_t t1,
                                                  uint2* __restrict__ seeds, uint2* __restrict__ z0,
                                                  uint2* __restrict__ z1, uint2* __restrict__ z2, AxCtl* ctl,
                                                  unsigned long long* __restrict__ work) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t K = (uint64_t)F.K, units = (t1 - t0) * K;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint2* const zq[3] = {z0, z1, z2};
  uint64_t ws = 0;
  for (uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull; w0 < units; w0 += nthr) {
    const uint64_t u = w0 + lane;
    const bool valid = u < units;
    const uint64_t ti = t0 + (valid ? u / K : 0);
    const int a1 = valid ? (int)(u % K) : 0;
    bool seeded = false, whole = false;
    uint32_t key0 = 0, direct = 0;
    if (valid) {
      uint32_t len, rc;
      const uint8_t* p = ax_pattern<FIXED, STRANDS>(pat, offs, lens, fixed_len, ti, len, rc);
      if (len >= (uint32_t)K) {
        PatWindow P;
        P.reset(p);
        key0 = rc ? kmer_key_rc(F.K, P, p, len) : kmer_key(F.K, P, p, len);
        seeded = true;
        whole = len == (uint32_t)K;
      }
      if (a1 == 0) {
        seeds[ti - t0] = seeded ? ax_lookup(F, key0) : make_uint2(0u, (uint32_t)F.N);
        if (WORK && seeded) ws += 1 + 3 * K + 9 * K * (K - 1) / 2 + (KMAX == 3 ? 27 * K * (K - 1) * (K - 2) / 6 : 0);
      }
    }
    auto emit = [&](bool act, uint32_t key, int tfrom, int lvl) {
      uint64_t pm = (act && seeded) ? ax_present_from(F, key, tfrom) : 0ull;
      if (whole) { direct += ax_sizes(F, key, tfrom, pm); pm = 0; }
      unsigned long long at = warp_reserve(&ctl->z[lvl], (uint32_t)__popcll(pm));
      for (; pm; pm &= pm - 1) zq[lvl][at++] = make_uint2((uint32_t)ti, ax_variant(key, tfrom, __ffsll((long long)pm) - 1));
    };
    emit(a1 == 0, key0, 0, KMAX - 1);                     // one substitution (the task's a1 = 0 thread)
    for (uint32_t r1 = 1; r1 < 4; ++r1) {
      const uint32_t k1 = kmer_subst(key0, a1, r1);
      emit(true, k1, a1 + 1, KMAX - 2);                   // two: the first at a1
      if (KMAX == 3)
        for (int a2 = 1; a2 < F.K; ++a2)
          for (uint32_t r2 = 1; r2 < 4; ++r2) emit(a2 > a1, kmer_subst(k1, a2, r2), a2 + 1, 0);   // three
    }
    if (valid && direct) atomicAdd(ax_out<STRANDS>(out, out_rc, ti), direct);
  }
  if (WORK && ws) { atomicAdd(work, (unsigned long long)ws); atomicAdd(work + 1, (unsigned long long)ws); }
}

// Warp-uniform refill of the lanes without a task from a range of indices [0, total) taken in
// chunks of FM_CHUNK from a global counter (as in k_fm_count).  Returns false once the range is
// exhausted and no lane holds a task.
struct AxRefill {
  uint64_t cb = 0, ce = 0;
  bool exhausted = false;
  template <class Seed>
  __device__ __forceinline__ bool run(bool& has, uint64_t total, unsigned long long* ctr, Seed&& seed) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t needm = __ballot_sync(0xffffffffu, !has);
    if (needm && !exhausted) {
      const uint32_t cnt = __popc(needm), r = __popc(needm & ((1u << lane) - 1u));
      const uint64_t avail = ce - cb;
      uint64_t nb = 0, ne = 0;
      if (cnt > avail) {
        if (lane == 0) nb = atomicAdd(ctr, (unsigned long long)FM_CHUNK);
        nb = __shfl_sync(0xffffffffu, nb, 0);
        ne = nb + FM_CHUNK < total ? nb + FM_CHUNK : total;
        if (nb >= total) { exhausted = true; nb = ne = total; }
      }
      if (!has) {
        const uint64_t t = r < avail ? cb + r : nb + (r - avail);
        if (r < avail || t < ne) { seed(t); has = true; }
      }
      if (cnt > avail) {
        const uint64_t take = cnt - avail;
        cb = nb + take < ne ? nb + take : ne;
        ce = ne;
      } else {
        cb += cnt;
      }
    }
    return !(exhausted && __ballot_sync(0xffffffffu, has) == 0);
  }
};

// The recursive one-substitution walk of an interval (the queue-overflow path of level-1 items).
template <int BW, bool WORK, class W>
__device__ __noinline__ uint32_t ax1_inline(const FmParams& F, W& P, int64_t j, uint32_t lo, uint32_t hi,
                                            FmWork& wk) {
  const uint4 C4 = __ldg(reinterpret_cast<const uint4*>(F.Ct));
  const uint32_t Cs[4] = {C4.x, C4.y, C4.z, C4.w};
  uint32_t total = 0;
  for (; j >= 0 && lo < hi; --j) {
    uint32_t ol[4], oh[4];
    fm_occ4_pair<BW, WORK>(F, lo, hi, ol, oh, wk);
    const uint32_t cj = P.at(j);
    uint32_t bl[4], bh[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      bl[c] = Cs[c] + ol[c];
      bh[c] = Cs[c] + oh[c];
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if ((uint32_t)c != cj && bl[c] < bh[c])
        total += j == 0 ? bh[c] - bl[c] : fm_continue<BW, WORK>(F, P, j - 1, bl[c], bh[c], wk);
    lo = sel4(bl, cj);
    hi = sel4(bh, cj);
  }
  return total + (lo < hi ? hi - lo : 0u);
}

// 3 CTAs per SM (80 registers, no spills): +5.6% on configs[3], +1.6% on the 150-bp reads over 4
// (64 registers, ~190 B of spills; profiles/r02_approx1_bfs_minb.txt)
#ifndef QR_AX1_PATH_MINB
#define QR_AX1_PATH_MINB 3
#endif
// SRC 0: the chunk's tasks from their seed intervals (level k, the only item of its task: the
// output is updated in place); 1: lookup items (task, key); 2: interval items (task, pos, lo, hi).
template <bool FIXED, int BW, int STRANDS, bool WORK, int SRC, int CHILD>   // CHILD: the children's mm
__global__ void __launch_bounds__(256, QR_AX1_PATH_MINB) k_ax_path(FmParams F, const uint8_t* __restrict__ pat,
                                                    const uint64_t* __restrict__ offs,
                                                    const uint32_t* __restrict__ lens, uint32_t fixed_len,
                                                    uint32_t* __restrict__ out, uint32_t* __restrict__ out_rc,
                                                    uint64_t t0, uint64_t t1, const uint2* __restrict__ seeds,
                                                    const void* __restrict__ items, const unsigned long long* n_items,
                                                    uint64_t items_cap, uint4* __restrict__ oq,
                                                    unsigned long long* oq_n, uint64_t oq_cap,
                                                    unsigned long long* ctr, unsigned long long* __restrict__ work) {
  FmWork wk;
  if (BW == 1) x2_masks_init();
  else qd_masks_init();
  const uint4 C4 = __ldg(reinterpret_cast<const uint4*>(F.Ct));
  const uint32_t Cs[4] = {C4.x, C4.y, C4.z, C4.w};
  const uint32_t lane = threadIdx.x & 31u;
  uint64_t total_items = t1 - t0;
  if (SRC != 0) {
    const unsigned long long nq = *n_items;
    total_items = nq < items_cap ? nq : items_cap;
  }
  StrandWindow<STRANDS> P;
  uint64_t ti = 0;
  uint32_t lo = 0, hi = 0, total = 0;
  int32_t j = -1;
  bool has = false;
  AxRefill rf;
  auto seed = [&](uint64_t t) {
    uint32_t len, rc;
    if (SRC == 0) {
      ti = t0 + t;
      const uint8_t* p = ax_pattern<FIXED, STRANDS>(pat, offs, lens, fixed_len, ti, len, rc);
      P.reset(p, len, rc);
      const uint2 iv = seeds[t];
      lo = iv.x; hi = iv.y;
      j = (int32_t)len - 1 - ((F.K && len >= (uint32_t)F.K) ? F.K : 0);
    } else if (SRC == 1) {
      const uint2 it = reinterpret_cast<const uint2*>(items)[t];
      ti = it.x;
      const uint8_t* p = ax_pattern<FIXED, STRANDS>(pat, offs, lens, fixed_len, ti, len, rc);
      P.reset(p, len, rc);
      const uint2 iv = ld_kmer(F.kmer + it.y);
      lo = iv.x; hi = iv.y;
      j = (int32_t)len - 1 - F.K;
    } else {
      const uint4 it = reinterpret_cast<const uint4*>(items)[t];
      ti = it.x;
      const uint8_t* p = ax_pattern<FIXED, STRANDS>(pat, offs, lens, fixed_len, ti, len, rc);
      P.reset(p, len, rc);
      lo = it.z; hi = it.w;
      j = (int32_t)it.y - 1;
    }
    total = 0;
  };
  while (rf.run(has, total_items, ctr, seed)) {
    // children in registers (static indices and selects: dynamically indexed arrays go to the stack)
    uint32_t bl[4] = {0u, 0u, 0u, 0u}, bh[4] = {0u, 0u, 0u, 0u}, em = 0;   // em: children to queue
    int32_t jc = 0;
    if (has) {
      if (j >= 0 && lo < hi) {
        uint32_t ol[4], oh[4];
        fm_occ4_pair<BW, WORK>(F, lo, hi, ol, oh, wk);
        const uint32_t cj = P.at(j);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          bl[c] = Cs[c] + ol[c];
          bh[c] = Cs[c] + oh[c];
          if ((uint32_t)c != cj && bl[c] < bh[c]) {
            if (j == 0) total += bh[c] - bl[c];           // substitution at P[0]: a leaf
            else em |= 1u << c;
          }
        }
        jc = j;
        lo = sel4(bl, cj);
        hi = sel4(bh, cj);
        --j;
      }
    }
    // the warp's new interval items (0..3 per lane): one atomic per warp that has any
    const uint32_t n = __popc(em);
    if (__ballot_sync(0xffffffffu, n != 0)) {
      const uint32_t lt = (1u << lane) - 1u;
      const uint32_t b0 = __ballot_sync(0xffffffffu, n & 1u), b1 = __ballot_sync(0xffffffffu, (n >> 1) & 1u);
      const uint32_t tot = __popc(b0) + 2u * __popc(b1);
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(oq_n, (unsigned long long)tot);
      base = __shfl_sync(0xffffffffu, base, 0) + __popc(b0 & lt) + 2u * __popc(b1 & lt);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if ((em >> c) & 1u) {
          const uint64_t at = base + __popc(em & ((1u << c) - 1u));
          if (at < oq_cap) oq[at] = make_uint4((uint32_t)ti, (uint32_t)jc, bl[c], bh[c]);
          else if (CHILD == 0) total += fm_continue<BW, WORK>(F, P, (int64_t)jc - 1, bl[c], bh[c], wk);
          else if (CHILD == 1) total += ax1_inline<BW, WORK>(F, P, (int64_t)jc - 1, bl[c], bh[c], wk);
          // CHILD 2 (k = 3): the queue holds 3 (len - K) items per task, every child fits
        }
    }
    if (has && !(j >= 0 && lo < hi)) {                   // finished: the item's exact count + leaves
      if (lo < hi) total += hi - lo;
      uint32_t* o = ax_out<STRANDS>(out, out_rc, ti);
      if (SRC == 0) *o += total;
      else if (total) atomicAdd(o, total);
      has = false;
    }
  }
  if (WORK && wk.ws) {
    atomicAdd(work, (unsigned long long)wk.ws);
    atomicAdd(work + 1, (unsigned long long)wk.wl);
  }
}

// Items with no substitution left: exact backward search of P[pos-1 .. 0].  LOOKUP: items
// (task, key) of k_ax_seed, the interval read from the table at refill (resolving them in
// k_ax_seed instead measured 1.35x slower on configs[3] at k = 1: its lanes then walk 3K
// dependent lookups, and the queue doubles); else (task, pos, lo, hi) of k_ax_path.
#ifndef QR_AX_CONT_MINB
#define QR_AX_CONT_MINB QR_APPROX1_MINB
#endif
template <bool FIXED, int BW, int STRANDS, bool WORK, bool LOOKUP>
__global__ void __launch_bounds__(256, QR_AX_CONT_MINB) k_ax_cont(FmParams F, const uint8_t* __restrict__ pat,
                                                    const uint64_t* __restrict__ offs,
                                                    const uint32_t* __restrict__ lens, uint32_t fixed_len,
                                                    uint32_t* __restrict__ out, uint32_t* __restrict__ out_rc,
                                                    const void* __restrict__ items, const unsigned long long* n_items,
                                                    uint64_t cap, unsigned long long* ctr,
                                                    unsigned long long* __restrict__ work) {
  FmWork wk;
  if (BW == 1) x2_masks_init();
  const unsigned long long nq = *n_items;
  const uint64_t total_items = nq < cap ? nq : cap;
  StrandWindow<STRANDS> P;
  uint64_t ti = 0;
  uint32_t lo = 0, hi = 0;
  int32_t j = -1;
  bool has = false;
  AxRefill rf;
  auto seed = [&](uint64_t t) {
    uint32_t len, rc;
    if (LOOKUP) {
      const uint2 it = reinterpret_cast<const uint2*>(items)[t];
      ti = it.x;
      const uint8_t* p = ax_pattern<FIXED, STRANDS>(pat, offs, lens, fixed_len, ti, len, rc);
      P.reset(p, len, rc);
      const uint2 iv = ld_kmer(F.kmer + it.y);
      lo = iv.x; hi = iv.y;
      j = (int32_t)len - 1 - F.K;
    } else {
      const uint4 it = reinterpret_cast<const uint4*>(items)[t];
      ti = it.x;
      const uint8_t* p = ax_pattern<FIXED, STRANDS>(pat, offs, lens, fixed_len, ti, len, rc);
      P.reset(p, len, rc);
      lo = it.z; hi = it.w;
      j = (int32_t)it.y - 1;
    }
  };
  while (rf.run(has, total_items, ctr, seed)) {
    if (has) {
      if (j >= 0 && lo < hi) {
        uint32_t nl;
        fm_step_cont<BW>(F, P.at(j), lo, hi, nl);
        if (WORK) { wk.ws += 1; wk.wl += nl; }
        --j;
      }
      if (!(j >= 0 && lo < hi)) {
        if (lo < hi) atomicAdd(ax_out<STRANDS>(out, out_rc, ti), hi - lo);
        has = false;
      }
    }
  }
  if (WORK && wk.ws) {
    atomicAdd(work, (unsigned long long)wk.ws);
    atomicAdd(work + 1, (unsigned long long)wk.wl);
  }
}

__global__ void k_u32_to_u64(const uint32_t* __restrict__ a, uint64_t* __restrict__ b, uint64_t m) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

static FmParams params_of(const qr_fm* fm) {
  FmParams F;
  F.lines = fm->bwt->lines;
  F.super = fm->bwt->super;
  F.kmer = fm->kmer;
  F.K = fm->kmer_k;
  F.spos = fm->spos;
  F.N = fm->N;
  F.last_line = fm->bwt->n_lines - 1;
  for (int c = 0; c < 4; ++c) F.C[c] = (uint32_t)fm->C[c];
  F.Ct = reinterpret_cast<const uint32_t*>(fm->kmer + kmer_c_offset(fm->kmer_k));
  F.spack = fm->bwt->spack;
  F.bw = fm->bwt->layout == QR_LAYOUT_QUADRANK16X2 ? 1 : 0;
  F.spack_half = (uint32_t)fm->bwt->spack_half;
  F.n_super = (uint32_t)fm->bwt->n_super;
  F.kbits = nullptr;
  return F;
}

// The approximate-search kernels' table (C[0..3] stays at the main table's tail, F.Ct).  When the
// build asked for a wider one than the count's (qr_fm_build's default from n = 2^24: 14, 2 GiB —
// each extra symbol of width replaces a level of the search tree by a lookup: configs[3] k = 2
// 29.4 / 35.1 / 38.3 M patterns/s and 150-bp reads 4.63 / 5.19 / 6.24 M reads/s at 12 / 13 / 14,
// profiles/r02_approx_width.jsonl) it is built here on the first approximate call, on the
// caller's stream, once, under a process-wide lock; the handle's pointers are read under it too.
static std::mutex g_ax_mu;
void fm_copy_locked(const qr_fm* src, qr_fm* dst) {
  std::lock_guard<std::mutex> g(g_ax_mu);
  *dst = *src;
}
extern int g_fm_kbits;
extern int g_fm_ax_bfs;
int g_fm_ax_bfs2 = 1;   // k = 2 breadth first too (knob fm_ax_bfs2)
int g_fm_ax_bfs3 = 1;   // k = 3 breadth first in auto mode (L2-resident BWT, fixed-length batches; knob
                        // fm_ax_bfs3): configs[3] 4.49 -> 6.90 M patterns/s, QuadRank16x2 5.25 -> 5.56 M
                        // (profiles/r02_approx_bfs_k3_ab.txt; with one seed thread per task 3.61: too few threads)
static qr_status fm_params_ax(const qr_fm* fmc, cudaStream_t st, FmParams& F) {
  qr_fm* fm = const_cast<qr_fm*>(fmc);                     // a lazily filled cache of the handle
  std::lock_guard<std::mutex> g(g_ax_mu);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) { cudaGetLastError(); cap = cudaStreamCaptureStatusNone; }
  // inside a CUDA-graph capture the build (allocation + synchronisation) cannot run: the captured
  // call uses the table the handle has now (results are width-independent)
  if (cap == cudaStreamCaptureStatusNone && fm->kmer_k_ax != fm->kmer_k_ax_want && fm->kmer_k_ax_want > 0) {
    const uint64_t nx = kmer_entries(fm->kmer_k_ax_want);
    uint2* t = nullptr;
    if (cudaMalloc((void**)&t, nx * sizeof(uint2)) != cudaSuccess) {
      cudaGetLastError();
      fm->kmer_k_ax_want = fm->kmer_k_ax;                  // no memory for it: keep the count's table
    } else {
      FmParams Fx = F;
      Fx.K = fm->kmer_k_ax_want;
      if (F.bw) k_kmer_table<1><<<(unsigned)((nx + 255) / 256), 256, 0, st>>>(Fx, t);
      else      k_kmer_table<0><<<(unsigned)((nx + 255) / 256), 256, 0, st>>>(Fx, t);
      cudaError_t e = cudaGetLastError();
      if (!e) e = cudaStreamSynchronize(st);               // complete before any stream may use it
      if (e) { cudaFree(t); return cuda_fail(e, "k_kmer_table (approximate search)"); }
      fm->kmer_ax = t;
      fm->kmer_k_ax = fm->kmer_k_ax_want;
    }
  }
  F.kmer = fm->kmer_ax;
  F.K = fm->kmer_k_ax;
  // the presence bitmap (ax_lookup): auto = when the table is sparse, N < 4^K / 2
  const bool bits = F.K > 0 && (g_fm_kbits == 2 || (g_fm_kbits == 0 && 2 * fm->N < kmer_entries(F.K)));
  if (bits && cap == cudaStreamCaptureStatusNone && fm->kmer_bits_k != F.K) {
    if (fm->kmer_bits) { cudaFree(fm->kmer_bits); fm->kmer_bits = nullptr; fm->kmer_bits_k = 0; }
    const uint64_t nx = kmer_entries(F.K);
    uint32_t* b = nullptr;
    if (cudaMalloc((void**)&b, ((nx + 31) / 32) * sizeof(uint32_t)) != cudaSuccess) {
      cudaGetLastError();                                  // no memory for it: look every K-mer up
    } else {
      const unsigned grid = (unsigned)std::min<uint64_t>((nx + 255) / 256, 148ull * 64);
      k_kmer_bits<<<grid, 256, 0, st>>>(F.kmer, nx, b);
      cudaError_t e = cudaGetLastError();
      if (!e) e = cudaStreamSynchronize(st);
      if (e) { cudaFree(b); return cuda_fail(e, "k_kmer_bits (approximate search)"); }
      fm->kmer_bits = b;
      fm->kmer_bits_k = F.K;
    }
  }
  F.kbits = bits && fm->kmer_bits_k == F.K ? fm->kmer_bits : nullptr;
  return QR_OK;
}

extern int g_fm_blocks_per_sm;
extern int g_fm_lean;
extern int g_fm_refill;
extern int g_fm_packed;

int l2_bytes(int device);

// Step flavour: the lean step issues fewer instructions but more L1 wavefronts and L2 requests
// (no line de-duplication); it wins when the BWT layout is L2-resident (instruction bound,
// configs[3]: 4.55 -> 5.53 G patterns/s) and loses when it is HBM-resident (request bound,
// configs[4]: 0.81 -> 0.76).  Auto = lean iff the layout fits in half of the L2.
static bool bwt_l2_resident(const qr_fm* fm) {
  return fm->bwt->n_lines * 64 <= (uint64_t)l2_bytes(fm->bwt->device) / 2;
}
// 1: de-duplicating step, 2: lean step, 3: one line per iteration (fm_step_pend; with the dynamic
// order and seeds: k_fm_count_l2).  Auto: 3 on L2-resident BWTs (configs[3]: 7.07 -> 8.68 G
// patterns/s over QuadRank16, 8.45 -> 9.12 over QuadRank16x2), 1 on HBM-resident ones (request-
// bound there: configs[4] 0.97 vs 0.86 with 3; profiles/r02_fm_step_probe.jsonl).
// On an HBM-resident BWT both strands at once (the paper's read workload) take the lean step
// with the seed pre-pass: 150-bp reads 0.533 -> 0.588 G reads/s, while one strand keeps the
// de-duplicating step without it (configs[4] 0.96 vs 0.89 / 0.95; profiles/r02_fm_hbm_strands.log).
static int fm_step_of(const qr_fm* fm, bool both) {
  if (g_fm_lean >= 1 && g_fm_lean <= 4) return g_fm_lean;
  return bwt_l2_resident(fm) ? 3 : both ? 2 : 1;
}

extern int g_fm_smem;

// Shared-memory superblock mode of the count kernel: the raw array when it fits the per-CTA
// budget that keeps 4 CTAs per SM (configs[3]: 18.7 KB), else the packed table if it does, else
// global memory (knob "fm_smem": 0 off, 1 auto (default), 2 the packed table whenever it fits a CTA).
constexpr uint64_t FM_SMEM_BUDGET = 48 * 1024;
static int fm_smem_mode(const qr_fm* fm, size_t* bytes) {
  const qr_index* b = fm->bwt;
  const uint64_t raw = b->n_super * 16, packed = super_pack_cta_bytes(b) * 2;
  *bytes = 0;
  if (g_fm_smem == 0) return 0;
  if (g_fm_smem == 1) {
    if (raw <= FM_SMEM_BUDGET) { *bytes = raw; return 1; }
    if (b->spack && packed <= FM_SMEM_BUDGET) { *bytes = packed; return 2; }
    return 0;
  }
  if (b->spack && packed + 1024 <= 227 * 1024) { *bytes = packed; return 2; }
  return 0;
}

// fixed-length batches whose post-seed symbols fit one u64 (2 bits each) take packed seeds
static bool fm_packable(const FmParams& F, uint32_t fixed_len) {
  if (g_fm_packed == 0) return false;
  const uint32_t kused = (F.K && fixed_len >= (uint32_t)F.K) ? (uint32_t)F.K : 0u;
  return fixed_len - kused <= 32u && fixed_len <= 46u;     // the seed kernel's 128-bit window
}

static int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

template <bool FIXED, bool WORK, int STRANDS, int STEP, int SMS>
static void launch_fm1(unsigned g, size_t smem, cudaStream_t st, const FmParams& F, const uint8_t* pat,
                       const uint64_t* offs, const uint32_t* lens, uint32_t fixed_len, uint32_t* out, uint32_t* out_rc,
                       uint64_t m, unsigned long long* w, unsigned long long* ctr, int sms, uint2* seeds) {
  if (ctr && seeds && STEP == 3) {
    const bool packed = FIXED && fm_packable(F, fixed_len);
    auto kern = packed ? (F.bw ? k_fm_count_l2<FIXED, WORK, STRANDS, SMS, 1, true> : k_fm_count_l2<FIXED, WORK, STRANDS, SMS, 0, true>)
                       : (F.bw ? k_fm_count_l2<FIXED, WORK, STRANDS, SMS, 1, false> : k_fm_count_l2<FIXED, WORK, STRANDS, SMS, 0, false>);
    if (packed)
      k_fm_seed_packed<STRANDS><<<grid_stride_blocks(m * STRANDS, 256, sms, 16), 256, 0, st>>>(F, pat, fixed_len, m,
                                                                                               (uint4*)seeds);
    else
      k_fm_seed<FIXED, STRANDS><<<grid_stride_blocks(m * STRANDS, 256, sms, 16), 256, 0, st>>>(F, pat, offs, lens,
                                                                                             fixed_len, m, seeds);
    smem_limit_raise((const void*)kern, smem, cur_device());
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem) != cudaSuccess || per_sm <= 0) {
      cudaGetLastError();
      per_sm = 1;
    }
    const uint64_t need = (m * STRANDS + 255) / 256;
    unsigned gp = (unsigned)((uint64_t)per_sm * sms < need ? (uint64_t)per_sm * sms : (need ? need : 1));
    // refill threshold: 8 idle lanes over QuadRank16, 4 over QuadRank16x2 (its shorter step makes
    // idle lanes cost less than refills): configs[3] 9.48 / 9.97 G patterns/s, knob fm_refill
    const uint32_t refill = g_fm_refill ? (uint32_t)g_fm_refill : (F.bw ? 4u : 8u);
    kern<<<gp, 256, smem, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, m, w, ctr, seeds, refill);
  } else if (ctr) {
    // QuadRank16x2 BWT: the sector-shared step, or the one-sector-per-iteration step (STEP 3)
    auto kern = F.bw ? k_fm_count<FIXED, WORK, STRANDS, STEP == 3 ? 3 : 0, SMS, true, 1>
                     : k_fm_count<FIXED, WORK, STRANDS, STEP, SMS, true, 0>;
    if (seeds)
      k_fm_seed<FIXED, STRANDS><<<grid_stride_blocks(m * STRANDS, 256, sms, 16), 256, 0, st>>>(F, pat, offs, lens,
                                                                                             fixed_len, m, seeds);
    smem_limit_raise((const void*)kern, smem, cur_device());
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem) != cudaSuccess || per_sm <= 0) {
      cudaGetLastError();
      per_sm = 1;
    }
    const uint64_t need = (m * STRANDS + 255) / 256;     // no more CTAs than tasks / 256
    unsigned gp = (unsigned)((uint64_t)per_sm * sms < need ? (uint64_t)per_sm * sms : (need ? need : 1));
    kern<<<gp, 256, smem, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, m, w, ctr, seeds);
  } else {
    auto kern = F.bw ? k_fm_count<FIXED, WORK, STRANDS, STEP == 3 ? 3 : 0, SMS, false, 1>
                     : k_fm_count<FIXED, WORK, STRANDS, STEP, SMS, false, 0>;
    smem_limit_raise((const void*)kern, smem, cur_device());
    kern<<<g, 256, smem, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, m, w, nullptr, nullptr);
  }
}

template <bool FIXED, bool WORK, int STRANDS, int STEP>
static void launch_fm2(int sms_mode, unsigned g, size_t smem, cudaStream_t st, const FmParams& F, const uint8_t* pat,
                       const uint64_t* offs, const uint32_t* lens, uint32_t fixed_len, uint32_t* out, uint32_t* out_rc,
                       uint64_t m, unsigned long long* w, unsigned long long* ctr, int sms, uint2* seeds) {
  if (sms_mode == 1)      launch_fm1<FIXED, WORK, STRANDS, STEP, 1>(g, smem, st, F, pat, offs, lens, fixed_len, out, out_rc, m, w, ctr, sms, seeds);
  else if (sms_mode == 2) launch_fm1<FIXED, WORK, STRANDS, STEP, 2>(g, smem, st, F, pat, offs, lens, fixed_len, out, out_rc, m, w, ctr, sms, seeds);
  else                    launch_fm1<FIXED, WORK, STRANDS, STEP, 0>(g, 0, st, F, pat, offs, lens, fixed_len, out, out_rc, m, w, ctr, sms, seeds);
}

extern int g_fm_dyn;
extern int g_fm_seed;

// Keep up to 2 GiB of freed stream-ordered allocations in the device's default pool (its default
// release threshold of 0 returns them to the driver at every synchronisation, so a per-call
// scratch buffer would be re-mapped on every call).
static void keep_pool_memory(int device, cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return;                                  // not during a capture (a device-wide setting)
  }
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> g(mu);
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = 2ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done[device] = true;
}

template <bool FIXED, bool WORK>
static cudaError_t launch_fm(const qr_fm* fm, int step, unsigned g, cudaStream_t st, const FmParams& F,
                             const uint8_t* pat, const uint64_t* offs, const uint32_t* lens, uint32_t fixed_len,
                             uint32_t* out, uint32_t* out_rc, uint64_t m, unsigned long long* w) {
  size_t smem = 0;
  const int sm = fm_smem_mode(fm, &smem);
  CounterLease lease;
  unsigned long long* ctr = nullptr;
  uint2* seeds = nullptr;
  cudaError_t e;
  if (g_fm_dyn) {
    // seed pre-pass: pays when the search is instruction-bound (L2-resident BWT: configs[3] 6.57
    // -> 7.21 G patterns/s) and for both strands at once (two seeds per pattern read), costs for
    // one strand when latency-bound (HBM: configs[4] 0.99 -> 0.86 in round 1, 0.96 -> 0.95 now)
    const bool pre = g_fm_seed == 2 || (g_fm_seed == 0 && (bwt_l2_resident(fm) || out_rc));
    if (pre) {
      keep_pool_memory(fm->bwt->device, st);
      // 16 B per task: room for the packed seeds (k_fm_seed_packed) when the batch qualifies
      if ((e = cudaMallocAsync((void**)&seeds, m * (out_rc ? 2 : 1) * sizeof(uint4), st))) return e;
    }
    if ((e = lease.acquire(fm->bwt->device, st, &ctr))) { if (seeds) cudaFreeAsync(seeds, st); return e; }
  }
  const int sms = fm->bwt->sm_count;
#define QR_FM_GO(S)                                                                                              \
  do {                                                                                                           \
    if (out_rc) launch_fm2<FIXED, WORK, 2, S>(sm, g, smem, st, F, pat, offs, lens, fixed_len, out, out_rc, m, w, ctr, sms, seeds); \
    else        launch_fm2<FIXED, WORK, 1, S>(sm, g, smem, st, F, pat, offs, lens, fixed_len, out, out_rc, m, w, ctr, sms, seeds); \
  } while (0)
  if (step == 3) QR_FM_GO(3);
  else if (step == 2) QR_FM_GO(2);
  else if (step == 4) QR_FM_GO(4);
  else QR_FM_GO(1);
#undef QR_FM_GO
  e = cudaGetLastError();
  if (ctr) {
    cudaError_t e2 = lease.release(st);
    if (!e) e = e2;
  }
  if (seeds) cudaFreeAsync(seeds, st);
  return e;
}

template <typename Kern>
static unsigned resident_grid(Kern k, int sms, size_t smem = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, smem) != cudaSuccess || per_sm <= 0) {
    cudaGetLastError();
    per_sm = 1;
  }
  return (unsigned)per_sm * (unsigned)sms;
}

// k = 1..3 breadth first (k_ax_*), tasks in chunks so that the queues stay within ~1.5 GB of the
// stream-ordered pool: the lookup items of the seed variants (exactly 3K, 9 C(K,2), 27 C(K,3) per
// task at most), the level-(k-1) interval items of the seed paths (k = 3: exactly 3 (len - K) per
// task, fixed-length batches only) and ~4 interval items per task for the levels below, whose
// overflow the emitting lane searches itself.
int g_ax_seed_split = 1;          // k = 2: seed variants over (task, a1) threads (knob fm_ax_seed_split)
uint64_t g_ax1_aq_per_task = 4;   // interval items per task and level (tests: 0 sends every one inline)
template <bool FIXED, int STRANDS, bool WORK, int KMAX>
static cudaError_t launch_ax_bfs(const qr_fm* fm, cudaStream_t st, const FmParams& F, const uint8_t* pat,
                                 const uint64_t* offs, const uint32_t* lens, uint32_t fixed_len, uint32_t* out,
                                 uint32_t* out_rc, uint64_t m, unsigned long long* work) {
  const uint64_t ntask = m * STRANDS;
  const uint64_t K = F.K > 0 ? (uint64_t)F.K : 0;
  const uint64_t nsub[4] = {1, 3 * K, 9 * K * (K ? K - 1 : 0) / 2, 27 * K * (K > 1 ? K - 1 : 0) * (K > 2 ? K - 2 : 0) / 6};
  uint64_t z_pt[3] = {0, 0, 0}, q_pt[3] = {0, 0, 0};
  for (int lvl = 0; lvl < KMAX; ++lvl) {
    z_pt[lvl] = nsub[KMAX - lvl];                         // level lvl holds the (KMAX - lvl)-substitution K-mers
    q_pt[lvl] = g_ax1_aq_per_task;
  }
  if (KMAX == 3) q_pt[2] = 3ull * (fixed_len > K ? fixed_len - K : 0);   // exact: no inline k = 2 walk
  uint64_t per_task = 8;
  for (int lvl = 0; lvl < KMAX; ++lvl) per_task += z_pt[lvl] * 8 + q_pt[lvl] * 16;
  uint64_t chunk = (3ull << 29) / per_task;
  chunk = chunk < 1024 ? 1024 : chunk;
  chunk = ntask < chunk ? ntask : chunk;
  size_t off = 256 + chunk * 8;
  size_t z_off[3] = {0, 0, 0}, q_off[3] = {0, 0, 0};
  for (int lvl = 0; lvl < KMAX; ++lvl) { z_off[lvl] = off; off += chunk * z_pt[lvl] * 8; }
  off = (off + 255) & ~(size_t)255;                       // uint4 items: 16-B aligned
  for (int lvl = 0; lvl < KMAX; ++lvl) { q_off[lvl] = off; off += chunk * q_pt[lvl] * 16; }
  keep_pool_memory(fm->bwt->device, st);
  unsigned char* buf = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&buf, off + 16, st);
  if (e) return e;
  AxCtl* ctl = reinterpret_cast<AxCtl*>(buf);
  uint2* seeds = reinterpret_cast<uint2*>(buf + 256);
  uint2* z[3];
  uint4* q[3];
  for (int lvl = 0; lvl < 3; ++lvl) {
    z[lvl] = reinterpret_cast<uint2*>(buf + z_off[lvl]);
    q[lvl] = reinterpret_cast<uint4*>(buf + q_off[lvl]);
  }
  const int sms = fm->bwt->sm_count;
#define QR_AX_K(KERN, ...) (F.bw ? KERN<FIXED, 1, STRANDS, WORK, __VA_ARGS__> : KERN<FIXED, 0, STRANDS, WORK, __VA_ARGS__>)
  auto kp_seed = QR_AX_K(k_ax_path, 0, (KMAX > 1 ? KMAX - 1 : 0));
  auto kp_z1 = QR_AX_K(k_ax_path, 1, 0);
  auto kp_q1 = QR_AX_K(k_ax_path, 2, 0);
  auto kp_z2 = QR_AX_K(k_ax_path, 1, 1);
  auto kp_q2 = QR_AX_K(k_ax_path, 2, 1);
  auto kcz = QR_AX_K(k_ax_cont, true);
  auto kcq = QR_AX_K(k_ax_cont, false);
#undef QR_AX_K
  const unsigned gp = resident_grid(kp_seed, sms), gc = resident_grid(kcz, sms);
  for (uint64_t t0 = 0; t0 < ntask && !e; t0 += chunk) {
    const uint64_t t1 = t0 + chunk < ntask ? t0 + chunk : ntask, nt = t1 - t0;
    if ((e = cudaMemsetAsync(ctl, 0, sizeof(AxCtl), st))) break;
    if (KMAX == 3 || (KMAX == 2 && g_ax_seed_split && K > 0)) {
      k_ax_zero<STRANDS><<<grid_stride_blocks(nt, 256, sms, 8), 256, 0, st>>>(out, out_rc, t0, t1);
      k_ax_seed3<FIXED, STRANDS, (KMAX == 3 ? 3 : 2), WORK><<<grid_stride_blocks(nt * K, 256, sms, 8), 256, 0, st>>>(
          F, pat, offs, lens, fixed_len, out, out_rc, t0, t1, seeds, z[0], z[1], z[2], ctl, work);
    } else {
      k_ax_seed<FIXED, STRANDS, KMAX, WORK><<<grid_stride_blocks(nt, 256, sms, 8), 256, 0, st>>>(
          F, pat, offs, lens, fixed_len, out, out_rc, t0, t1, seeds, z[0], z[1], z[2], ctl, work);
    }
    // the seed paths (level KMAX), then each level's lookup and interval items down to level 1
    kp_seed<<<gp, 256, 0, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, t0, t1, seeds, nullptr, nullptr, 0,
                                q[KMAX - 1], &ctl->q[KMAX - 1], nt * q_pt[KMAX - 1], &ctl->ctr[0], work);
    for (int lvl = KMAX - 1; lvl >= 1; --lvl) {
      auto kz = lvl == 2 ? kp_z2 : kp_z1;
      auto kq = lvl == 2 ? kp_q2 : kp_q1;
      kz<<<gp, 256, 0, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, t0, t1, nullptr, z[lvl], &ctl->z[lvl],
                             nt * z_pt[lvl], q[lvl - 1], &ctl->q[lvl - 1], nt * q_pt[lvl - 1], &ctl->ctr[2 * lvl],
                             work);
      kq<<<gp, 256, 0, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, t0, t1, nullptr, q[lvl], &ctl->q[lvl],
                             nt * q_pt[lvl], q[lvl - 1], &ctl->q[lvl - 1], nt * q_pt[lvl - 1],
                             &ctl->ctr[2 * lvl + 1], work);
    }
    kcz<<<gc, 256, 0, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, z[0], &ctl->z[0], nt * z_pt[0], &ctl->ctr[7], work);
    kcq<<<gc, 256, 0, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, q[0], &ctl->q[0], nt * q_pt[0], &ctl->ctr[8], work);
    e = cudaGetLastError();
  }
  cudaError_t e2 = cudaFreeAsync(buf, st);
  return e ? e : e2;
}

template <bool FIXED, int STRANDS, bool WORK>
static cudaError_t launch_approx_s(const qr_fm* fm, unsigned g, cudaStream_t st, const FmParams& F, const uint8_t* pat,
                                   const uint64_t* offs, const uint32_t* lens, uint32_t fixed_len, uint32_t* out,
                                   uint32_t* out_rc, uint64_t m, int kmax, unsigned long long* work) {
  // breadth first (auto, profiles/r02_approx_bfs_k2_ab.txt, r02_approx_bfs_k3_ab.txt): k = 1
  // everywhere but on an L2-resident QuadRank16x2 BWT (150-bp reads 52.8 -> 103 M reads/s,
  // configs[3] 1.31 -> 1.48 G; QuadRank16x2 configs[3] 1.68 recursive vs 1.50); k = 2, 3 on
  // L2-resident BWTs (configs[3] k = 2 69.9 -> 88.3 M, k = 3 4.49 -> 6.90 M; QuadRank16x2 91.0 ->
  // 93.2 M, 5.25 -> 5.56 M; the reads, HBM-resident, k = 2 6.98 recursive vs 6.11)
  const bool l2 = bwt_l2_resident(fm);
  const bool bfs = g_fm_ax_bfs == 2 ||
                   (g_fm_ax_bfs == 1 && (kmax == 1 ? !(F.bw == 1 && l2) : l2 && (kmax == 2 ? g_fm_ax_bfs2 : g_fm_ax_bfs3)));
  if (bfs && g_fm_dyn && m * STRANDS < (1ull << 32)) {
    if (kmax == 1) return launch_ax_bfs<FIXED, STRANDS, WORK, 1>(fm, st, F, pat, offs, lens, fixed_len, out, out_rc, m, work);
    if (kmax == 2) return launch_ax_bfs<FIXED, STRANDS, WORK, 2>(fm, st, F, pat, offs, lens, fixed_len, out, out_rc, m, work);
    if (kmax == 3 && FIXED && F.K > 0 && (g_fm_ax_bfs == 2 || g_fm_ax_bfs3))
      return launch_ax_bfs<FIXED, STRANDS, WORK, 3>(fm, st, F, pat, offs, lens, fixed_len, out, out_rc, m, work);
  }
  auto kern = kmax == 1 ? (F.bw ? k_fm_approx1<FIXED, 1, STRANDS, WORK> : k_fm_approx1<FIXED, 0, STRANDS, WORK>)
            : kmax == 2 ? (F.bw ? k_fm_approxk<FIXED, 1, 2, STRANDS, WORK> : k_fm_approxk<FIXED, 0, 2, STRANDS, WORK>)
                        : (F.bw ? k_fm_approxk<FIXED, 1, 3, STRANDS, WORK> : k_fm_approxk<FIXED, 0, 3, STRANDS, WORK>);
  // k >= 2: the backtracking frames in shared memory (FmFrames), 256 threads x WORDS u32
  const size_t smem = kmax == 2 ? FmFrames<2>::WORDS * 256 * 4 : kmax == 3 ? FmFrames<3>::WORDS * 256 * 4 : 0;
  smem_limit_raise((const void*)kern, smem, cur_device());
  if (!g_fm_dyn) {
    kern<<<g, 256, smem, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, m, nullptr, work);
    return cudaGetLastError();
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem) != cudaSuccess || per_sm <= 0) {
    cudaGetLastError();
    per_sm = 1;
  }
  const unsigned res = (unsigned)per_sm * (unsigned)fm->bwt->sm_count;
  CounterLease lease;
  unsigned long long* ctr = nullptr;
  cudaError_t e = lease.acquire(fm->bwt->device, st, &ctr);
  if (e) return e;
  kern<<<res < g ? res : g, 256, smem, st>>>(F, pat, offs, lens, fixed_len, out, out_rc, m, ctr, work);
  e = cudaGetLastError();
  cudaError_t e2 = lease.release(st);
  return e ? e : e2;
}

template <bool FIXED>
static cudaError_t launch_approx(const qr_fm* fm, unsigned g, cudaStream_t st, const FmParams& F, const uint8_t* pat,
                                 const uint64_t* offs, const uint32_t* lens, uint32_t fixed_len, uint32_t* out,
                                 uint32_t* out_rc, uint64_t m, int kmax, unsigned long long* work) {
  if (work) {
    if (out_rc) return launch_approx_s<FIXED, 2, true>(fm, g, st, F, pat, offs, lens, fixed_len, out, out_rc, m, kmax, work);
    return launch_approx_s<FIXED, 1, true>(fm, g, st, F, pat, offs, lens, fixed_len, out, nullptr, m, kmax, work);
  }
  if (out_rc) return launch_approx_s<FIXED, 2, false>(fm, g, st, F, pat, offs, lens, fixed_len, out, out_rc, m, kmax, nullptr);
  return launch_approx_s<FIXED, 1, false>(fm, g, st, F, pat, offs, lens, fixed_len, out, nullptr, m, kmax, nullptr);
}

qr_status fm_count_device(const qr_fm* fm, const uint8_t* pat, const uint32_t* lengths, uint32_t fixed_len,
                          uint32_t* out, uint32_t* out_rc, uint64_t m, uint64_t* work, cudaStream_t st, int approx) {
  if (m == 0) return QR_OK;
  FmParams F = params_of(fm);
  const int sms = fm->bwt->sm_count;
  const uint64_t tasks = out_rc ? 2 * m : m;
  unsigned g = grid_stride_blocks(tasks, 256, sms, g_fm_blocks_per_sm);
  unsigned long long* w = reinterpret_cast<unsigned long long*>(work);
  cudaError_t e;
  FmParams Fa = F;
  if (approx) {
    qr_status sa = fm_params_ax(fm, st, Fa);
    if (sa != QR_OK) return sa;
  }
  if (!lengths) {
    if (approx) e = launch_approx<true>(fm, g, st, Fa, pat, nullptr, nullptr, fixed_len, out, out_rc, m, approx, w);
    else if (work) e = launch_fm<true, true>(fm, fm_step_of(fm, out_rc != nullptr), g, st, F, pat, nullptr, nullptr, fixed_len, out, out_rc, m, w);
    else      e = launch_fm<true, false>(fm, fm_step_of(fm, out_rc != nullptr), g, st, F, pat, nullptr, nullptr, fixed_len, out, out_rc, m, w);
    if (e) return cuda_fail(e, "k_fm_count");
    return QR_OK;
  }
  uint64_t* offs = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  if ((e = cudaMallocAsync((void**)&offs, m * 8, st))) return cuda_fail(e, "alloc offsets");
  k_u32_to_u64<<<grid_stride_blocks(m, 256, sms, 8), 256, 0, st>>>(lengths, offs, m);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, offs, offs, (int64_t)m, st))) { cudaFreeAsync(offs, st); return cuda_fail(e, "scan"); }
  if ((e = cudaMallocAsync(&tmp, tb, st))) { cudaFreeAsync(offs, st); return cuda_fail(e, "alloc scan tmp"); }
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, offs, offs, (int64_t)m, st))) {
    cudaFreeAsync(offs, st); cudaFreeAsync(tmp, st); return cuda_fail(e, "scan");
  }
  if (approx) e = launch_approx<false>(fm, g, st, Fa, pat, offs, lengths, 0, out, out_rc, m, approx, w);
  else if (work) e = launch_fm<false, true>(fm, fm_step_of(fm, out_rc != nullptr), g, st, F, pat, offs, lengths, 0, out, out_rc, m, w);
  else      e = launch_fm<false, false>(fm, fm_step_of(fm, out_rc != nullptr), g, st, F, pat, offs, lengths, 0, out, out_rc, m, w);
  cudaFreeAsync(offs, st);
  cudaFreeAsync(tmp, st);
  if (e) return cuda_fail(e, "k_fm_count");
  return QR_OK;
}

// d_text: device copy, >= ceil(n/32) words, zero padded.  d_sa: optional device SA (N u32).
qr_status fm_build_device(const uint64_t* d_text, uint64_t n, const uint32_t* d_sa_given, int device, cudaStream_t st,
                          qr_fm** out, int kmer_k, int bwt_layout, int kmer_k_ax) {
  const uint64_t N = n + 1;
  const int sms = sm_count(device);
  cudaError_t e;
  uint32_t* d_sa = nullptr;
  uint64_t* d_bwt = nullptr;
  unsigned long long* d_aux = nullptr;   // [0] spos, [1..4] symbol counts
  unsigned long long h_aux[5];
  qr_fm* fm = new (std::nothrow) qr_fm();
  if (!fm) return fail(QR_ENOMEM, "qr_fm_build: host allocation");
  // build temporaries: plain cudaMalloc (see build_sa), freed after the stream is drained
  auto release = [&]() {
    cudaStreamSynchronize(st);
    cudaFree(d_sa); cudaFree(d_bwt); cudaFree(d_aux);
    d_sa = nullptr; d_bwt = nullptr; d_aux = nullptr;
  };
  auto bail = [&](qr_status s) {
    release();
    qr_fm_free(fm);
    return s;
  };
  const uint64_t L = N / QD_B + 1;
  const uint64_t Lx = N / Q16X2_B + 1;
  const uint64_t bwt_words = 7 * L > 6 * Lx ? 7 * L : 6 * Lx;   // words the QuadRank16 / 16x2 builders read
  if ((e = cudaMalloc((void**)&d_aux, 5 * 8))) return bail(cuda_fail(e, "alloc aux"));
  cudaMemsetAsync(d_aux, 0, 5 * 8, st);
  if (!d_sa_given) {
    if ((e = cudaMalloc((void**)&d_sa, N * 4))) return bail(cuda_fail(e, "alloc sa"));
    qr_status s = build_sa(d_text, n, sms, st, d_sa);
    if (s != QR_OK) return bail(s);
  }
  if ((e = cudaMalloc((void**)&d_bwt, bwt_words * 8))) return bail(cuda_fail(e, "alloc bwt"));
  cudaMemsetAsync(d_bwt, 0, bwt_words * 8, st);
  k_bwt<<<grid_stride_blocks((N + 31) / 32, 256, sms, 16), 256, 0, st>>>(d_text, d_sa_given ? d_sa_given : d_sa, N,
                                                                          d_bwt, d_aux);
  k_sym_counts<<<grid_stride_blocks((n + 31) / 32, 256, sms, 8), 256, 0, st>>>(d_text, n, d_aux + 1);
  if ((e = cudaGetLastError())) return bail(cuda_fail(e, "k_bwt"));
  qr_status s = bwt_layout == QR_LAYOUT_QUADRANK16X2 ? quadrank16x2_build_device(d_bwt, N, device, st, &fm->bwt)
                                                     : quadrank_build_device(d_bwt, N, device, st, &fm->bwt);
  if (s != QR_OK) return bail(s);
  cudaMemcpyAsync(h_aux, d_aux, 5 * 8, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st))) return bail(cuda_fail(e, "fm build sync"));
  fm->n = n;
  fm->N = N;
  fm->spos = h_aux[0];
  fm->C[0] = 1;
  for (int c = 1; c < 4; ++c) fm->C[c] = fm->C[c - 1] + h_aux[c];   // C[c] = 1 + #{t_i < c}
  fm->C[4] = N;
  fm->kmer_k = kmer_k;
  const uint64_t ne = kmer_entries(kmer_k);
  if ((e = cudaMalloc((void**)&fm->kmer, (kmer_c_offset(kmer_k) + 2) * sizeof(uint2)))) return bail(cuda_fail(e, "alloc kmer"));
  {
    uint32_t Ch[4] = {(uint32_t)fm->C[0], (uint32_t)fm->C[1], (uint32_t)fm->C[2], (uint32_t)fm->C[3]};
    if ((e = cudaMemcpyAsync(fm->kmer + kmer_c_offset(kmer_k), Ch, sizeof(Ch), cudaMemcpyHostToDevice, st)))
      return bail(cuda_fail(e, "copy C"));
    if ((e = cudaStreamSynchronize(st))) return bail(cuda_fail(e, "copy C"));
  }
  FmParams F = params_of(fm);
  if (kmer_k) {
    if (F.bw) k_kmer_table<1><<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(F, fm->kmer);
    else      k_kmer_table<0><<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(F, fm->kmer);
  }
  if ((e = cudaGetLastError())) return bail(cuda_fail(e, "k_kmer_table"));
  fm->kmer_ax = fm->kmer;                                  // the approximate-search table: built
  fm->kmer_k_ax = kmer_k;                                  // on the first approximate call when
  fm->kmer_k_ax_want = kmer_k_ax > 0 ? kmer_k_ax : kmer_k; // wider than the count's (fm_params_ax)
  if ((e = cudaStreamSynchronize(st))) { release(); qr_fm_free(fm); return cuda_fail(e, "fm build"); }
  release();
  *out = fm;
  return QR_OK;
}

}  // namespace qr
