// qr_common.cuh — shared internals of libqrank.so (product path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "qrank.h"

namespace qr {

// ---- BiRank16 geometry (§3) ----
constexpr uint64_t BI_B = 496;          // data bits per 64-B line
constexpr uint32_t BI_SB_LOG = 7;       // 128 lines per superblock
constexpr uint32_t BI_SHIFT = 11;       // s_i = floor(rank(iS)/2^11)
constexpr uint32_t BI_ANCHOR = 240;     // b_j to data bit 240 = line bit 256
constexpr uint64_t BI_MAX_N = 1ull << 43;
constexpr uint64_t Q16X2_B = 192;       // QuadRank16x2: 2 sectors x 96 chars (B200 sector-local variant)
constexpr uint64_t B32X2_B = 448;       // BiRank32x2: 2 sectors x 224 data bits
constexpr uint32_t B32X2_SB_LOG = 23;   // 2^23 lines per L1 entry: deltas < 2^23 * 448 + 336 < 2^32
constexpr uint64_t B16X2_B = 480;       // BiRank16x2: 2 sectors x 240 data bits

// ---- QuadRank16 geometry (§4, Listing 1) ----
constexpr uint64_t QD_B = 224;          // data chars per line
constexpr uint32_t QD_SB_LOG = 8;       // 256 lines per superblock, PAPER.md:511 (reading R5)
constexpr uint32_t QD_SHIFT = 13;
constexpr uint32_t QD_ANCHOR = 96;      // data char 96 = line char 128
constexpr uint64_t QD_MAX_N = 1ull << 45;

// ---- launch geometry ----
constexpr int NUM_SMS_B200 = 148;

}  // namespace qr

// Handle layouts (opaque to callers).
struct qr_index {
  int sigma;            // 2 or 4
  int layout;           // QR_LAYOUT_* (include/qrank.h)
  int device;
  uint64_t n;           // text length (bits or symbols)
  uint64_t n_lines;     // floor(n/B)+1
  uint64_t n_super;     // ((n_lines-1) >> SB_LOG) + 1
  uint4* lines;         // n_lines * 64 B, 256-B aligned (cudaMalloc)
  uint32_t* super;      // sigma=2: u32[n_super]; sigma=4: u32[4*n_super] (s_{i,c} at 4i+c)
  int sm_count;
  uint64_t* spack;      // superblock array re-encoded for the shared-memory rank kernels (sbcache.cu), or null
  uint64_t spack_half;  // groups held by each CTA of the 2-CTA cluster
  uint64_t* spack_big = nullptr;   // BiRank16 n >= 2^35: 5-superblock groups over a CS-CTA cluster (sbcache.cu)
  uint64_t spack_big_slots = 0;    // groups per CTA
  uint32_t spack_big_cs = 0;       // cluster size (4, 8 or 16)
  uint32_t spack_big_hi[3] = {};   // BiRank16: first group whose base s >> 24 is >= 1, 2, 3
};

struct qr_fm {
  qr_index* bwt;        // QuadRank16 over the N = n+1 BWT symbols ('$' stored as A)
  uint64_t n;           // text length
  uint64_t N;           // n + 1
  uint64_t spos;        // BWT row of '$'
  uint64_t C[5];        // C[c] = 1 + #{t_i < c}; C[4] = N
  uint2* kmer;          // 4^K [lo, hi) intervals after K backward steps, then C[0..3] (2 uint2)
  int kmer_k;           // K: table of K-mers (PAPER.md:918 uses 8; 0 = no table)
  uint2* kmer_ax;       // the approximate-search kernels' table (== kmer unless a wider one pays there)
  int kmer_k_ax;
  int kmer_k_ax_want;   // its width; a wider table than kmer_k is built on the first approximate call
  uint32_t* kmer_bits;  // presence bitmap of kmer_ax (bit key = its interval is non-empty), or null
  int kmer_bits_k;      // the width it was built for (0: none)
};

namespace qr {
// thread-local error channel
void set_error(const char* fmt, ...);
qr_status fail(qr_status st, const char* fmt, ...);
qr_status cuda_fail(cudaError_t e, const char* what);

// pointer space: 0 = host (pinned or pageable), 1 = device on `device`, -1 = device elsewhere
int pointer_space(const void* p, int device);

// SM count of a device (cached)
int sm_count(int device);
// number of q[i] > n into *cnt (device u64, accumulated): the opt-in range check (QR_ERANGE)
cudaError_t launch_count_gt(const uint64_t* q, uint64_t m, uint64_t n, unsigned long long* cnt, int device,
                            cudaStream_t st);
// Raise a kernel's dynamic shared-memory limit on `device` to at least `bytes` (process-wide,
// mutex-guarded, never lowers it: a later launch with a smaller size must not undercut a
// concurrent or cached launch that needs more).  Returns the attribute call's error, if any.
cudaError_t smem_limit_raise(const void* kern, size_t bytes, int device);

// internal builders used by fm.cu
qr_status quadrank_build_device(const uint64_t* d_text2b, uint64_t n, int device, cudaStream_t st, qr_index** out);
qr_status alloc_index(int sigma, uint64_t n, int device, qr_index** out, int layout = 0);
uint64_t super_bytes_of(const qr_index* h);
qr_status birank64x2_build_device(const uint64_t* d_bits, uint64_t n, int device, cudaStream_t st, qr_index** out);
qr_status birank16x2_build_device(const uint64_t* d_bits, uint64_t n, int device, cudaStream_t st, qr_index** out);
cudaError_t launch_b16x2_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                              int what, cudaStream_t st);
qr_status birank32x2_build_device(const uint64_t* d_bits, uint64_t n, int device, cudaStream_t st, qr_index** out);
cudaError_t launch_b32x2_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                              int what, cudaStream_t st);
qr_status quadrank16x2_build_device(const uint64_t* d_text, uint64_t n, int device, cudaStream_t st, qr_index** out);
cudaError_t launch_q16x2_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                              int what, cudaStream_t st);
qr_status quadrank64_build_device(const uint64_t* d_text, uint64_t n, int device, cudaStream_t st, qr_index** out);
cudaError_t launch_rank_chain(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                              uint64_t chain_len, cudaStream_t st);
cudaError_t launch_variant(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m, int what,
                           cudaStream_t st);

// kernel launchers (device pointers; validated by api.cu)
cudaError_t launch_birank_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                               cudaStream_t st);
cudaError_t launch_quadrank_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                 cudaStream_t st);
cudaError_t launch_quadrank_all4(const qr_index* h, const uint64_t* q, uint64_t* out4, uint64_t m, cudaStream_t st);
cudaError_t launch_gather(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode, cudaStream_t st);
inline uint64_t kmer_entries(int k) { return 1ull << (2 * k); }
// C[0..3] (16 B) follow the table at an even entry index, so that the 16-B load is aligned
inline uint64_t kmer_c_offset(int k) { return (kmer_entries(k) + 1) & ~1ull; }
qr_status fm_count_device(const qr_fm* fm, const uint8_t* pat, const uint32_t* lengths, uint32_t fixed_len,
                          uint32_t* out, uint32_t* out_rc, uint64_t m, uint64_t* work, cudaStream_t st,
                          int approx = 0);
cudaError_t launch_big_pack_qd(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                               int what, cudaStream_t st);
cudaError_t launch_big_pack_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                 cudaStream_t st);
qr_status build_super_pack(qr_index* h, cudaStream_t st);
uint64_t super_pack_cta_bytes(const qr_index* h);
int super_pack_clusters(const qr_index* h);
enum { RANK_LANE = 0, RANK_PAIR = 1, RANK_CLUSTER = 2 };
int rank_shape(const qr_index* h, uint64_t m);
cudaError_t launch_lane_table_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                   int what, cudaStream_t st);
cudaError_t launch_super_pack_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                                   int what, cudaStream_t st);
qr_status birank_build_device(const uint64_t* d_bits, uint64_t n, int device, cudaStream_t st, qr_index** out);

// A zeroed work counter (4 u64 words) for one launch of a dynamic-work-order kernel
// (counters.cu).  acquire() before the launch, release() after it, on the same stream; the
// lease holds a host lock in between.
struct CounterLease {
  void* ring = nullptr;
  uint32_t slot = 0;
  unsigned long long* own = nullptr;   // graph-capture path: a stream-ordered allocation
  cudaError_t acquire(int device, cudaStream_t st, unsigned long long** ctr);
  cudaError_t release(cudaStream_t st);
  ~CounterLease();
};

// grid for a grid-stride kernel: a multiple of the SM count
inline unsigned grid_stride_blocks(uint64_t work_items, unsigned threads, int sms, int blocks_per_sm) {
  uint64_t need = (work_items + threads - 1) / threads;
  uint64_t cap = (uint64_t)sms * (uint64_t)blocks_per_sm;
  if (need > cap) need = cap;
  return need ? (unsigned)need : 1u;
}

// ---- device helpers ----
// 256-bit gather of one 32-B sector (LDG.E.256 on sm_100a), not allocated in L1, with the
// L2 fill limited to the 64-B line that holds it (.L2::64B: without it every random miss
// fills a whole 128-B L2 line — 123 B of DRAM per load measured by ncu, tools/gather_probe).
// Deliberately not .nc: ptxas may sink .nc loads below later uses (it did, serialising the K
// queries of a thread); a coherent load cannot move past the stores that follow the gathers.
__device__ __forceinline__ void ld_sector_na(const void* p, uint64_t& w0, uint64_t& w1, uint64_t& w2, uint64_t& w3) {
  asm volatile("ld.global.L1::no_allocate.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3)
               : "l"(p));
}
// Same, allocating in L1 (FM: lo and hi of a step, and consecutive steps, often share a line).
__device__ __forceinline__ void ld_sector(const void* p, uint64_t& w0, uint64_t& w1, uint64_t& w2, uint64_t& w3) {
  asm volatile("ld.global.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w0), "=l"(w1), "=l"(w2), "=l"(w3) : "l"(p));
}
// One k-mer table entry of the approximate search (8 B at a random index of a table of up to
// 2 GiB), read-only, not allocated in L1, L2 fill limited to its 64-B line: __ldg's default 128-B
// fill read 4 DRAM sectors per lookup (ncu: 3.6e9 sectors for 8.6e8 lookups + 2.9e8 BWT steps at
// k = 2); +11% / +12% / +20% patterns/s at k = 1 / 2 / 3 (profiles/r02_kmer_ld.log).  The exact
// count's seed lookups keep __ldg: its table is L2-resident and the hinted load measured -6% there.
// (An L2::evict_first policy on top, to shield the BWT's lines, measured no better.)
__device__ __forceinline__ uint2 ld_kmer(const uint2* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
// Predicated 8-byte read-only load (no branch: lanes with pred == 0 issue nothing and get 0).
__device__ __forceinline__ uint64_t ldg_u64_if(bool pred, const void* p) {
  uint64_t v;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\tmov.u64 %0, 0;\n\t@q ld.global.nc.u64 %0, [%1];\n\t}"
      : "=l"(v)
      : "l"(p), "r"((uint32_t)pred));
  return v;
}
// Predicated 8-byte read-only load into v (v keeps its value where pred == 0; no branch).
__device__ __forceinline__ void ldg_u64_keep(bool pred, const void* p, uint64_t& v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u64 %0, [%1];\n\t}"
               : "+l"(v)
               : "l"(p), "r"((uint32_t)pred));
}
// ~0 << d with the PTX clamp (d = 64 gives 0; C's shift would be undefined there)
__device__ __forceinline__ uint64_t ones_shl(uint32_t d) {
  uint64_t v;
  asm("shl.b64 %0, %1, %2;" : "=l"(v) : "l"(~0ull), "r"(d));
  return v;
}
// Query-stream loads (coalesced, read once).  Coherent + volatile so that the software
// prefetch of the next group's queries stays where it is written (issued while the current
// group's gathers are in flight) instead of being sunk to its use.
__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_stream_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.global.L1::no_allocate.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_stream_v4u64(uint64_t* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.L1::no_allocate.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
               : "memory");
}

// prefix mask of the first x bits of word t of a multi-word field (x may exceed the word).
__device__ __forceinline__ uint64_t prefix_mask(int x, int t) {
  int d = x - 64 * t;
  d = d < 0 ? 0 : d;
  return d >= 64 ? ~0ull : ((1ull << d) - 1ull);
}

}  // namespace qr
