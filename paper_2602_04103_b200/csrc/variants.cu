// variants.cu — the paper's no-L1-array layout variants on sm_100a (NEXT §8(f)4).
//
// On B200 a random query costs L2 requests, not bytes: BiRank16/QuadRank16
// need a second request per query for the L2-resident superblock word.  The paper's larger
// variants that "completely remove the L1 level" trade space for exactly that request:
//
// BiRank64x2 (33.3%): every 32-B sector is self-contained —
//   sector h of line j = [u64 v_{j,h} | 192 data bits],  v_{j,h} = rank(384 j + 192 h + 96),
//   i.e. two 64-bit values "to 1/4th and 3/4th" of the 384-bit block (the x2 family anchors,
//   PAPER.md:484-492).  Line j's data bits are text words [6j, 6j+6) (384 = 6 * 64).  A query
//   reads ONE 32-B sector: one L2 request, no superblock word, popcount over <= 96 bits.
//
// QuadRank64 (100%, "stores 4 64-bit values, as does BWA-MEM, removing the
//   L1 array ... each half is now only 64 of them"): sector 0 = v_{j,c} = rank(128 j + 64, c)
//   for c = A, C, G, T; sector 1 = 128 chars as two transposed negated plane pairs (word 4+2t =
//   NOT low bits, 5+2t = NOT high bits of chars 64t..64t+63).  Line j's chars are text words
//   [4j, 4j+4).  A query needs both sectors: the lane pair loads them in one instruction (one
//   L2 request), no superblock word.
#include <cub/device/device_scan.cuh>

#include "qr_common.cuh"
#include "sched.cuh"

namespace qr {

extern int g_rank_k;
extern int g_rank_blocks_per_sm;

__device__ __forceinline__ uint64_t even_bits64(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return x;
}

// ------------------------------------------------------------------ BiRank64x2 build

// per sector: total and count of its first 96 data bits
__global__ void k_b64_count(const uint64_t* __restrict__ t, uint64_t L, uint64_t* __restrict__ tot,
                            uint32_t* __restrict__ half) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t* w = t + 6 * j + 3 * h;
      const uint32_t a = __popcll(w[0]), b = __popcll(w[1] & 0xffffffffull);
      half[2 * j + h] = a + b;
      tot[2 * j + h] = a + __popcll(w[1]) + __popcll(w[2]);
    }
  }
}

__global__ void k_b64_write(const uint64_t* __restrict__ t, uint64_t L, const uint64_t* __restrict__ R,
                            const uint32_t* __restrict__ half, uint4* __restrict__ lines) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(lines + 4 * j);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t* w = t + 6 * j + 3 * h;
      const uint64_t v = R[2 * j + h] + half[2 * j + h];      // rank(384 j + 192 h + 96)
      dst[2 * h] = make_ulonglong2(v, w[0]);
      dst[2 * h + 1] = make_ulonglong2(w[1], w[2]);
    }
  }
}

qr_status birank64x2_build_device(const uint64_t* d_bits, uint64_t n, int device, cudaStream_t st, qr_index** out) {
  qr_index* h = nullptr;
  qr_status rs = alloc_index(2, n, device, &h, QR_LAYOUT_BIRANK64X2);
  if (rs != QR_OK) return rs;
  const uint64_t L = h->n_lines;
  uint64_t *tot = nullptr, *R = nullptr;
  uint32_t* half = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t e;
  auto bail = [&](cudaError_t err, const char* what) {
    cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(half, st); cudaFreeAsync(tmp, st);
    qr_free(h);
    return cuda_fail(err, what);
  };
  if ((e = cudaMallocAsync((void**)&tot, 2 * L * 8, st))) return bail(e, "alloc tot");
  if ((e = cudaMallocAsync((void**)&R, 2 * L * 8, st))) return bail(e, "alloc R");
  if ((e = cudaMallocAsync((void**)&half, 2 * L * 4, st))) return bail(e, "alloc half");
  const unsigned g = grid_stride_blocks(L, 256, h->sm_count, 16);
  k_b64_count<<<g, 256, 0, st>>>(d_bits, L, tot, half);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, tot, R, (int64_t)(2 * L), st))) return bail(e, "scan size");
  if ((e = cudaMallocAsync(&tmp, tb, st))) return bail(e, "alloc scan tmp");
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, tot, R, (int64_t)(2 * L), st))) return bail(e, "scan");
  k_b64_write<<<g, 256, 0, st>>>(d_bits, L, R, half, h->lines);
  if ((e = cudaGetLastError())) return bail(e, "k_b64_write");
  cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(half, st); cudaFreeAsync(tmp, st);
  *out = h;
  return QR_OK;
}

// ------------------------------------------------------------------ BiRank16x2 build
// BiRank16x2 (6.72%): "stores two 16-bit deltas, to 1/4th and 3/4th into the
// block", so a query popcounts at most a quarter of the line.  B200 reading (R24):
// the two halves are the two 32-B sectors, each self-contained except for the superblock word:
//   sector h of line j = [u16 d_{j,h} | 240 data bits],  data bits [480 j + 240 h, +240),
//   d_{j,h} = rank(480 j + 240 h + 120) - 2^11 s_{j>>7},  s_i = floor(rank(128 i * 480) / 2^11)
// (128 lines per superblock as in BiRank16: d <= 127*480 + 360 + 2047 = 63,367 < 2^16).  Line
// j's data are text u16 words [30 j, 30 j + 30) (480 = 30 * 16); a query reads ONE sector.
__global__ void k_b16x2_count(const uint16_t* __restrict__ t16, uint64_t L, uint32_t* __restrict__ part,
                              uint64_t* __restrict__ tot) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint16_t* w = t16 + 30 * j;
    uint32_t c[30];
#pragma unroll
    for (int k = 0; k < 30; ++k) c[k] = __popc((uint32_t)w[k]);
    uint32_t a0 = __popc((uint32_t)w[7] & 0xffu), a1 = __popc((uint32_t)w[22] & 0xffu), h0 = 0, h1 = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) { a0 += c[k]; a1 += c[15 + k]; }
#pragma unroll
    for (int k = 0; k < 15; ++k) { h0 += c[k]; h1 += c[15 + k]; }
    part[2 * j] = a0;              // rank(240 h + 120) - rank(0) within the line, h = 0
    part[2 * j + 1] = h0 + a1;     // ... h = 1
    tot[j] = h0 + h1;
  }
}

__global__ void k_b16x2_write(const uint16_t* __restrict__ t16, uint64_t L, const uint64_t* __restrict__ R,
                              const uint32_t* __restrict__ part, uint4* __restrict__ lines, uint32_t* __restrict__ super) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t sb = R[(j >> BI_SB_LOG) << BI_SB_LOG] >> BI_SHIFT;
    if ((j & ((1u << BI_SB_LOG) - 1)) == 0) super[j >> BI_SB_LOG] = (uint32_t)sb;
    const uint16_t* w = t16 + 30 * j;
    uint4* dst = lines + 4 * j;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t d = (uint32_t)(R[j] + part[2 * j + h] - (sb << BI_SHIFT));
      uint32_t u[8];
      u[0] = d | ((uint32_t)w[15 * h] << 16);
#pragma unroll
      for (int k = 1; k < 8; ++k) u[k] = (uint32_t)w[15 * h + 2 * k - 1] | ((uint32_t)w[15 * h + 2 * k] << 16);
      dst[2 * h] = make_uint4(u[0], u[1], u[2], u[3]);
      dst[2 * h + 1] = make_uint4(u[4], u[5], u[6], u[7]);
    }
  }
}

qr_status birank16x2_build_device(const uint64_t* d_bits, uint64_t n, int device, cudaStream_t st, qr_index** out) {
  qr_index* h = nullptr;
  qr_status rs = alloc_index(2, n, device, &h, QR_LAYOUT_BIRANK16X2);
  if (rs != QR_OK) return rs;
  const uint64_t L = h->n_lines;
  uint64_t *tot = nullptr, *R = nullptr;
  uint32_t* part = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t e;
  auto bail = [&](cudaError_t err, const char* what) {
    cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(part, st); cudaFreeAsync(tmp, st);
    qr_free(h);
    return cuda_fail(err, what);
  };
  if ((e = cudaMallocAsync((void**)&tot, L * 8, st))) return bail(e, "alloc tot");
  if ((e = cudaMallocAsync((void**)&R, L * 8, st))) return bail(e, "alloc R");
  if ((e = cudaMallocAsync((void**)&part, 2 * L * 4, st))) return bail(e, "alloc part");
  const unsigned g = grid_stride_blocks(L, 256, h->sm_count, 16);
  const uint16_t* t16 = reinterpret_cast<const uint16_t*>(d_bits);
  k_b16x2_count<<<g, 256, 0, st>>>(t16, L, part, tot);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, tot, R, (int64_t)L, st))) return bail(e, "scan size");
  if ((e = cudaMallocAsync(&tmp, tb, st))) return bail(e, "alloc scan tmp");
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, tot, R, (int64_t)L, st))) return bail(e, "scan");
  k_b16x2_write<<<g, 256, 0, st>>>(t16, L, R, part, h->lines, h->super);
  if ((e = cudaGetLastError())) return bail(e, "k_b16x2_write");
  cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(part, st); cudaFreeAsync(tmp, st);
  if ((rs = build_super_pack(h, st)) != QR_OK) { qr_free(h); return rs; }
  *out = h;
  return QR_OK;
}

// ------------------------------------------------------------------ BiRank32x2 build
// BiRank32x2 (14.3%): "stores two 32-bit L2 values, shrinking the L1 array".
// B200 reading (R26): sector h of line j = [u32 d_{j,h} | 224 data bits 448 j + 224 h ..],
// d_{j,h} = rank(448 j + 224 h + 112) - L1[j >> 23], L1[i] = rank(2^23 * 448 * i) (u64): deltas
// stay below 2^23 * 448 + 336 < 2^32, and the L1 array (8 B per 3.76 G bits, 18.7 KB at n = 2^43)
// fits every CTA's shared memory.  Line j's data = text u32 words [14 j, 14 j + 14).
__global__ void k_b32x2_count(const uint32_t* __restrict__ t32, uint64_t L, uint32_t* __restrict__ part,
                              uint64_t* __restrict__ tot) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t* w = t32 + 14 * j;
    uint32_t c[14];
#pragma unroll
    for (int k = 0; k < 14; ++k) c[k] = __popc(w[k]);
    // anchors at data bits 112 and 336: words 0..2 + low 16 bits of word 3 (resp. 7..9 + word 10 low)
    uint32_t a0 = __popc(w[3] & 0xffffu), a1 = __popc(w[10] & 0xffffu), h0 = 0, h1 = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) { a0 += c[k]; a1 += c[7 + k]; }
#pragma unroll
    for (int k = 0; k < 7; ++k) { h0 += c[k]; h1 += c[7 + k]; }
    part[2 * j] = a0;
    part[2 * j + 1] = h0 + a1;
    tot[j] = h0 + h1;
  }
}

__global__ void k_b32x2_write(const uint32_t* __restrict__ t32, uint64_t L, const uint64_t* __restrict__ R,
                              const uint32_t* __restrict__ part, uint4* __restrict__ lines, uint64_t* __restrict__ l1) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t base = R[(j >> B32X2_SB_LOG) << B32X2_SB_LOG];
    if ((j & ((1ull << B32X2_SB_LOG) - 1)) == 0) l1[j >> B32X2_SB_LOG] = base;
    const uint32_t* w = t32 + 14 * j;
    uint4* dst = lines + 4 * j;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t d = (uint32_t)(R[j] + part[2 * j + h] - base);
      dst[2 * h] = make_uint4(d, w[7 * h], w[7 * h + 1], w[7 * h + 2]);
      dst[2 * h + 1] = make_uint4(w[7 * h + 3], w[7 * h + 4], w[7 * h + 5], w[7 * h + 6]);
    }
  }
}

qr_status birank32x2_build_device(const uint64_t* d_bits, uint64_t n, int device, cudaStream_t st, qr_index** out) {
  qr_index* h = nullptr;
  qr_status rs = alloc_index(2, n, device, &h, QR_LAYOUT_BIRANK32X2);
  if (rs != QR_OK) return rs;
  const uint64_t L = h->n_lines;
  uint64_t *tot = nullptr, *R = nullptr;
  uint32_t* part = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t e;
  auto bail = [&](cudaError_t err, const char* what) {
    cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(part, st); cudaFreeAsync(tmp, st);
    qr_free(h);
    return cuda_fail(err, what);
  };
  if ((e = cudaMallocAsync((void**)&tot, L * 8, st))) return bail(e, "alloc tot");
  if ((e = cudaMallocAsync((void**)&R, L * 8, st))) return bail(e, "alloc R");
  if ((e = cudaMallocAsync((void**)&part, 2 * L * 4, st))) return bail(e, "alloc part");
  const unsigned g = grid_stride_blocks(L, 256, h->sm_count, 16);
  const uint32_t* t32 = reinterpret_cast<const uint32_t*>(d_bits);
  k_b32x2_count<<<g, 256, 0, st>>>(t32, L, part, tot);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, tot, R, (int64_t)L, st))) return bail(e, "scan size");
  if ((e = cudaMallocAsync(&tmp, tb, st))) return bail(e, "alloc scan tmp");
  if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, tot, R, (int64_t)L, st))) return bail(e, "scan");
  k_b32x2_write<<<g, 256, 0, st>>>(t32, L, R, part, h->lines, reinterpret_cast<uint64_t*>(h->super));
  if ((e = cudaGetLastError())) return bail(e, "k_b32x2_write");
  cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(part, st); cudaFreeAsync(tmp, st);
  *out = h;
  return QR_OK;
}

// ------------------------------------------------------------------ QuadRank16x2 build
// QuadRank16x2 (B200 sector-local variant, NEXT §8(f)4, R25; 33.3%): the σ=4 analogue
// of BiRank16x2.  Each 32-B sector is self-contained except for the superblock words:
//   sector h of line j = [u16 d_{j,h,c} for c = A, C, G, T | 96 chars as transposed bit planes],
//   chars 192 j + 96 h .. +96 (text u64 words [6 j + 3 h, +3)): word 1 = low bits of chars 0..63,
//   word 2 = their high bits, word 3 = low bits of chars 64..95 | high bits << 32,
//   d_{j,h,c} = rank(192 j + 96 h + 48, c) - 2^13 s_{j>>8,c},  s_{i,c} = floor(rank(256 i 192, c)/2^13)
// (256 lines per superblock as QuadRank16: d <= 255*192 + 144 + 8191 = 57,295 < 2^16).  A query
// reads ONE sector for rank and for rank_4 and counts at most 48 characters.
__device__ __forceinline__ void q16x2_count_word(uint64_t w, uint64_t range, uint32_t (&a)[4]) {
  const uint64_t M = 0x5555555555555555ull & range;
  const uint64_t lo = w & M, hi = (w >> 1) & M;
  const uint32_t c3 = __popcll(lo & hi), l1 = __popcll(lo), h1 = __popcll(hi), len = __popcll(M);
  a[3] += c3; a[1] += l1 - c3; a[2] += h1 - c3; a[0] += len - l1 - h1 + c3;
}

// per line: counts to each sector's anchor (chars [0,48) and [0,144)) packed 8 bits x 4, and totals
__global__ void k_q16x2_count(const uint64_t* __restrict__ t, uint64_t L, uint64_t* __restrict__ tot,
                              uint32_t* __restrict__ part) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t* w = t + 6 * j;
    uint32_t a[4] = {0, 0, 0, 0};
    q16x2_count_word(w[0], ~0ull, a);
    q16x2_count_word(w[1], 0xffffffffull, a);                    // chars [32, 48)
    part[2 * j] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
    q16x2_count_word(w[1], ~0xffffffffull, a);
    q16x2_count_word(w[2], ~0ull, a);
    q16x2_count_word(w[3], ~0ull, a);
    q16x2_count_word(w[4], 0xffffffffull, a);                    // chars [128, 144)
    part[2 * j + 1] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);
    q16x2_count_word(w[4], ~0xffffffffull, a);
    q16x2_count_word(w[5], ~0ull, a);
#pragma unroll
    for (int c = 0; c < 4; ++c) tot[(uint64_t)c * L + j] = a[c];
  }
}

__global__ void k_q16x2_write(const uint64_t* __restrict__ t, uint64_t L, const uint64_t* __restrict__ R,
                              const uint32_t* __restrict__ part, uint4* __restrict__ lines, uint32_t* __restrict__ super) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j0 = (j >> QD_SB_LOG) << QD_SB_LOG;
    uint64_t sb[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      sb[c] = R[(uint64_t)c * L + j0] >> QD_SHIFT;
      if (j == j0) super[4 * (j >> QD_SB_LOG) + c] = (uint32_t)sb[c];
    }
    const uint64_t* w = t + 6 * j;
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(lines + 4 * j);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t pc = part[2 * j + h];
      uint64_t d = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        d |= (R[(uint64_t)c * L + j] + ((pc >> (8 * c)) & 0xffu) - (sb[c] << QD_SHIFT)) << (16 * c);
      const uint64_t a = w[3 * h], b = w[3 * h + 1], c2 = w[3 * h + 2];
      const uint64_t lo01 = even_bits64(a) | (even_bits64(b) << 32), hi01 = even_bits64(a >> 1) | (even_bits64(b >> 1) << 32);
      const uint64_t p2 = even_bits64(c2) | (even_bits64(c2 >> 1) << 32);
      dst[2 * h] = make_ulonglong2(d, lo01);
      dst[2 * h + 1] = make_ulonglong2(hi01, p2);
    }
  }
}

qr_status quadrank16x2_build_device(const uint64_t* d_text, uint64_t n, int device, cudaStream_t st, qr_index** out) {
  qr_index* h = nullptr;
  qr_status rs = alloc_index(4, n, device, &h, QR_LAYOUT_QUADRANK16X2);
  if (rs != QR_OK) return rs;
  const uint64_t L = h->n_lines;
  uint64_t *tot = nullptr, *R = nullptr;
  uint32_t* part = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t e;
  auto bail = [&](cudaError_t err, const char* what) {
    cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(part, st); cudaFreeAsync(tmp, st);
    qr_free(h);
    return cuda_fail(err, what);
  };
  if ((e = cudaMallocAsync((void**)&tot, 4 * L * 8, st))) return bail(e, "alloc tot");
  if ((e = cudaMallocAsync((void**)&R, 4 * L * 8, st))) return bail(e, "alloc R");
  if ((e = cudaMallocAsync((void**)&part, 2 * L * 4, st))) return bail(e, "alloc part");
  const unsigned g = grid_stride_blocks(L, 256, h->sm_count, 16);
  k_q16x2_count<<<g, 256, 0, st>>>(d_text, L, tot, part);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, tot, R, (int64_t)L, st))) return bail(e, "scan size");
  if ((e = cudaMallocAsync(&tmp, tb, st))) return bail(e, "alloc scan tmp");
  for (int c = 0; c < 4; ++c)
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, tot + (uint64_t)c * L, R + (uint64_t)c * L, (int64_t)L, st)))
      return bail(e, "scan");
  k_q16x2_write<<<g, 256, 0, st>>>(d_text, L, R, part, h->lines, h->super);
  if ((e = cudaGetLastError())) return bail(e, "k_q16x2_write");
  cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(part, st); cudaFreeAsync(tmp, st);
  if ((rs = build_super_pack(h, st)) != QR_OK) { qr_free(h); return rs; }
  *out = h;
  return QR_OK;
}

// ------------------------------------------------------------------ QuadRank64 build

__global__ void k_q64_count(const uint64_t* __restrict__ t, uint64_t L, uint64_t* __restrict__ tot,
                            uint32_t* __restrict__ c64) {
  const uint64_t M = 0x5555555555555555ull;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t a[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k == 2) c64[j] = a[0] | (a[1] << 8) | (a[2] << 16) | (a[3] << 24);   // chars [0,64)
      const uint64_t w = t[4 * j + k];
      const uint64_t lo = w & M, hi = (w >> 1) & M;
      const uint32_t c3 = __popcll(lo & hi), l1 = __popcll(lo), h1 = __popcll(hi);
      a[3] += c3; a[1] += l1 - c3; a[2] += h1 - c3; a[0] += 32 - l1 - h1 + c3;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) tot[(uint64_t)c * L + j] = a[c];
  }
}

__global__ void k_q64_write(const uint64_t* __restrict__ t, uint64_t L, const uint64_t* __restrict__ R,
                            const uint32_t* __restrict__ c64, uint4* __restrict__ lines) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < L; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t cp = c64[j];
    uint64_t v[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = R[(uint64_t)c * L + j] + ((cp >> (8 * c)) & 0xffu);   // rank(128j+64, c)
    const uint64_t* w = t + 4 * j;
    const uint64_t l0 = even_bits64(w[0]) | (even_bits64(w[1]) << 32), h0 = even_bits64(w[0] >> 1) | (even_bits64(w[1] >> 1) << 32);
    const uint64_t l1 = even_bits64(w[2]) | (even_bits64(w[3]) << 32), h1 = even_bits64(w[2] >> 1) | (even_bits64(w[3] >> 1) << 32);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(lines + 4 * j);
    dst[0] = make_ulonglong2(v[0], v[1]);
    dst[1] = make_ulonglong2(v[2], v[3]);
    dst[2] = make_ulonglong2(~l0, ~h0);
    dst[3] = make_ulonglong2(~l1, ~h1);
  }
}

qr_status quadrank64_build_device(const uint64_t* d_text, uint64_t n, int device, cudaStream_t st, qr_index** out) {
  qr_index* h = nullptr;
  qr_status rs = alloc_index(4, n, device, &h, QR_LAYOUT_QUADRANK64);
  if (rs != QR_OK) return rs;
  const uint64_t L = h->n_lines;
  uint64_t *tot = nullptr, *R = nullptr;
  uint32_t* c64 = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t e;
  auto bail = [&](cudaError_t err, const char* what) {
    cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(c64, st); cudaFreeAsync(tmp, st);
    qr_free(h);
    return cuda_fail(err, what);
  };
  if ((e = cudaMallocAsync((void**)&tot, 4 * L * 8, st))) return bail(e, "alloc tot");
  if ((e = cudaMallocAsync((void**)&R, 4 * L * 8, st))) return bail(e, "alloc R");
  if ((e = cudaMallocAsync((void**)&c64, L * 4, st))) return bail(e, "alloc c64");
  const unsigned g = grid_stride_blocks(L, 256, h->sm_count, 16);
  k_q64_count<<<g, 256, 0, st>>>(d_text, L, tot, c64);
  if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tb, tot, R, (int64_t)L, st))) return bail(e, "scan size");
  if ((e = cudaMallocAsync(&tmp, tb, st))) return bail(e, "alloc scan tmp");
  for (int c = 0; c < 4; ++c)
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, tb, tot + (uint64_t)c * L, R + (uint64_t)c * L, (int64_t)L, st)))
      return bail(e, "scan");
  k_q64_write<<<g, 256, 0, st>>>(d_text, L, R, c64, h->lines);
  if ((e = cudaGetLastError())) return bail(e, "k_q64_write");
  cudaFreeAsync(tot, st); cudaFreeAsync(R, st); cudaFreeAsync(c64, st); cudaFreeAsync(tmp, st);
  *out = h;
  return QR_OK;
}

// ------------------------------------------------------------------ queries

template <int K>
__device__ __forceinline__ void v_load_q(const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs, uint64_t i0,
                                         uint64_t stride, uint64_t m, uint64_t (&qn)[K], uint32_t (&cn)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint64_t idx = i0 + (uint64_t)k * stride;
    qn[k] = idx < m ? ld_stream_u64(q + idx) : 0;
    if (cs) cn[k] = idx < m ? ld_stream_u8(cs + idx) & 3u : 0u;
  }
}

// BiRank64x2: one lane per query, one 32-B sector.  Count over the sector's 192 data bits
// (3 words) of [x, 96) or [96, x): mask = prefix(x) XOR prefix(96), the symmetric difference.
template <int K, int MODE, bool DYN>   // MODE 0: rank; 1: gather ceiling (same load, no popcount)
__global__ void __launch_bounds__(256) k_b64_rank(const uint4* __restrict__ lines, const uint64_t* __restrict__ q,
                                                  const uint8_t* __restrict__ cs, uint64_t* __restrict__ out,
                                                  uint64_t m, uint64_t last_line, unsigned long long* ctr) {
  const uint32_t u = sc_unit_in_warp<32>();
  ScSched sc = sc_first<K, DYN, 32>(ctr);
  uint64_t qn[K];
  uint32_t cn[K];
  v_load_q<K>(q, cs, sc.gb + u, sc.stride, m, qn, cn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, nthr = sc.stride;
    uint64_t qq[K], w[K][4];
    uint32_t xx[K], cc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      qq[k] = qn[k];
      cc[k] = cn[k];
      uint64_t j = qq[k] < (1ull << 39) ? (uint64_t)((uint32_t)(qq[k] >> 7) / 3u) : qq[k] / 384;   // floor(q/384)
      j = j > last_line ? last_line : j;
      uint64_t r = qq[k] - j * 384;
      r = r > 383 ? 383 : r;
      const uint32_t h = r >= 192 ? 1u : 0u;
      xx[k] = (uint32_t)r - 192u * h;
      ld_sector_na(lines + 4 * j + 2 * h, w[k][0], w[k][1], w[k][2], w[k][3]);
    }
    sc = sc_next<K, DYN, 32>(sc, ctr);
    v_load_q<K>(q, cs, sc.gb + u, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * nthr;
      uint64_t r;
      if (MODE == 1) {
        r = w[k][0] ^ w[k][1] ^ w[k][2] ^ w[k][3];
      } else {
        const int x = (int)xx[k];
        uint32_t cnt = __popcll(w[k][1] & (prefix_mask(x, 0) ^ ~0ull)) +
                       __popcll(w[k][2] & (prefix_mask(x, 1) ^ 0xffffffffull)) +
                       __popcll(w[k][3] & prefix_mask(x, 2));
        r = x >= 96 ? w[k][0] + cnt : w[k][0] - cnt;
        if (cs && cc[k] == 0) r = qq[k] - r;                   // sigma = 2 with c = 0
      }
      if (idx < m) st_stream_u64(out + idx, r);
    }
  }
}

// QuadRank64: lane pairs (lane 0: sector 0 with the four counts, lane 1: sector 1 with the
// 128 chars) -> one request per query.  ALL4 = 1 returns the four ranks.
template <int K, int MODE, bool DYN>   // MODE 0: rank(q,c); 1: rank_4(q); 2: gather ceiling
__global__ void __launch_bounds__(256) k_q64_rank(const uint4* __restrict__ lines, const uint64_t* __restrict__ q,
                                                  const uint8_t* __restrict__ cs, uint64_t* __restrict__ out,
                                                  uint64_t m, uint64_t last_line, unsigned long long* ctr) {
  const uint32_t half = threadIdx.x & 1u;
  const uint32_t u = sc_unit_in_warp<16>();
  ScSched sc = sc_first<K, DYN, 16>(ctr);
  uint64_t qn[K];
  uint32_t cn[K];
  v_load_q<K>(q, MODE == 0 ? cs : nullptr, sc.gb + u, sc.stride, m, qn, cn);
  while (sc.gb < m) {
    const uint64_t i0 = sc.gb + u, npair = sc.stride;
    uint64_t qq[K], w[K][4];
    uint32_t cc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      qq[k] = qn[k];
      cc[k] = MODE == 0 ? cn[k] : 0u;
      uint64_t j = qq[k] >> 7;
      j = j > last_line ? last_line : j;
      ld_sector_na(lines + 4 * j + 2 * half, w[k][0], w[k][1], w[k][2], w[k][3]);
      if (j << 7 != (qq[k] & ~127ull)) qq[k] = (j << 7) | 127;   // q > n: clamp inside the last line
    }
    sc = sc_next<K, DYN, 16>(sc, ctr);
    v_load_q<K>(q, MODE == 0 ? cs : nullptr, sc.gb + u, sc.stride, m, qn, cn);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t idx = i0 + (uint64_t)k * npair;
      const uint32_t x = (uint32_t)(qq[k] & 127u);
      const bool right = x >= 64;
      const int y = (int)(x & 63u);
      const uint64_t msk = prefix_mask(y, 0) ^ (right ? 0ull : ~0ull);     // [y,64) of pair 0 or [0,y) of pair 1
      const uint64_t wl = right ? w[k][2] : w[k][0], wh = right ? w[k][3] : w[k][1];   // lane 1's plane pair
      if (MODE == 2) {
        uint64_t v = w[k][0] ^ w[k][1] ^ w[k][2] ^ w[k][3];
        v ^= __shfl_xor_sync(0xffffffffu, v, 1);
        if (half == 0 && idx < m) st_stream_u64(out + idx, v);
      } else if (MODE == 0) {
        const uint32_t c = cc[k];
        const uint64_t cl = 0ull - (uint64_t)(c & 1u), ch = 0ull - (uint64_t)(c >> 1);
        const uint32_t cnt = __popcll((wl ^ cl) & (wh ^ ch) & msk);
        const uint64_t vc = (c & 2u) ? ((c & 1u) ? w[k][3] : w[k][2]) : ((c & 1u) ? w[k][1] : w[k][0]);
        uint64_t v = half ? (right ? (uint64_t)cnt : 0ull - (uint64_t)cnt) : vc;
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (half == 0 && idx < m) st_stream_u64(out + idx, v);
      } else {
        const uint64_t l = ~wl & msk, hh = ~wh & msk;
        const uint32_t nl = __popcll(l), nh = __popcll(hh), nt = __popcll(l & hh);
        const uint32_t len = right ? (uint32_t)y : 64u - (uint32_t)y;
        const uint32_t packed = (len - nl - nh + nt) | ((nl - nt) << 8) | ((nh - nt) << 16) | (nt << 24);
        const uint32_t other = __shfl_xor_sync(0xffffffffu, packed, 1);
        if (half == 0 && idx < m) {
          uint64_t r[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t cn4 = (other >> (8 * c)) & 0xffu;
            r[c] = right ? w[k][c] + cn4 : w[k][c] - cn4;
          }
          st_stream_v4u64(out + 4 * idx, r[0], r[1], r[2], r[3]);
        }
      }
    }
  }
}

// persistent grid for the dynamic order: as many 256-thread CTAs as fit at once
template <typename Kern>
static unsigned resident_blocks(Kern kern, int sms) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess || per_sm <= 0) {
    cudaGetLastError();
    per_sm = 1;
  }
  return (unsigned)(per_sm * sms);
}

template <int K, bool DYN>
static void v_launch2(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m, int what,
                      unsigned long long* ctr, cudaStream_t st) {
  const uint64_t last = h->n_lines - 1;
  const bool b64 = h->layout == QR_LAYOUT_BIRANK64X2;
  // static order: a multi-wave grid sized from the work; dynamic: the resident grid (capped by the work)
  const uint64_t lanes = b64 ? (m + K - 1) / K : (2 * m + K - 1) / K;
  unsigned g = grid_stride_blocks(lanes, 256, h->sm_count, g_rank_blocks_per_sm);
  auto go = [&](auto kern, const uint8_t* cc) {
    unsigned gg = g;
    if (DYN) { const unsigned r = resident_blocks(kern, h->sm_count); gg = r < g ? r : g; }
    kern<<<gg, 256, 0, st>>>(h->lines, q, cc, out, m, last, ctr);
  };
  if (b64) {
    if (what == 2) go(k_b64_rank<K, 1, DYN>, nullptr);
    else           go(k_b64_rank<K, 0, DYN>, c);
  } else {
    if (what == 0)      go(k_q64_rank<K, 0, DYN>, c);
    else if (what == 1) go(k_q64_rank<K, 1, DYN>, nullptr);
    else                go(k_q64_rank<K, 2, DYN>, nullptr);
  }
}

template <int K>
static cudaError_t v_launch(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                            int what, cudaStream_t st) {
  if (!use_dyn_order(m)) {
    v_launch2<K, false>(h, q, c, out, m, what, nullptr, st);
    return cudaGetLastError();
  }
  CounterLease lease;
  unsigned long long* ctr = nullptr;
  cudaError_t e;
  if ((e = lease.acquire(h->device, st, &ctr))) return e;
  v_launch2<K, true>(h, q, c, out, m, what, ctr, st);
  e = cudaGetLastError();
  cudaError_t e2 = lease.release(st);
  return e ? e : e2;
}

// what: 0 = rank, 1 = rank_4 (QuadRank64), 2 = gather ceiling
cudaError_t launch_variant(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m, int what,
                           cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  if (h->layout == QR_LAYOUT_BIRANK16X2) return launch_b16x2_rank(h, q, c, out, m, what, st);
  if (h->layout == QR_LAYOUT_QUADRANK16X2) return launch_q16x2_rank(h, q, c, out, m, what, st);
  if (h->layout == QR_LAYOUT_BIRANK32X2) return launch_b32x2_rank(h, q, c, out, m, what, st);
  switch (g_rank_k) {
    case 1: return v_launch<1>(h, q, c, out, m, what, st);
    case 4: return v_launch<4>(h, q, c, out, m, what, st);
    case 8: return v_launch<8>(h, q, c, out, m, what, st);
    default: return v_launch<2>(h, q, c, out, m, what, st);
  }
}


// ------------------------------------------------------------------ latency (dependent-chain) mode
// The paper's "latency" benchmark mode (each query "dependent on the result of
// the previous one"; NEXT §8(f)4) with SPEC's chaining rule: within a chain of length L,
// the i-th query is q_eff = (q[i] + r_{i-1}) mod (n+1), r_{-1} = 0, and out[i] = rank(q_eff, c[i]).
// One thread per chain, one rank at a time: the time per step is the loaded latency of one
// random line gather (+ the superblock word), the GPU analogue of the paper's ~80 ns DRAM bound.
namespace {
struct RankOne {
  const qr_index h;
  __device__ __forceinline__ uint64_t operator()(uint64_t q, uint32_t c) const {
    const uint64_t last = h.n_lines - 1;
    uint64_t a[4], b[4] = {0, 0, 0, 0};
    if (h.layout == QR_LAYOUT_BIRANK16) {
      uint64_t j = q / BI_B;
      j = j > last ? last : j;
      uint64_t p = 16 + q - j * BI_B;
      p = p > 511 ? 511 : p;
      const uint4* ln = h.lines + 4 * j;
      ld_sector_na(ln, a[0], a[1], a[2], a[3]);
      if (p >= 256) ld_sector_na(ln + 2, b[0], b[1], b[2], b[3]);
      const uint32_t s = __ldg(h.super + (j >> BI_SB_LOG));
      const bool right = p >= 256;
      const int x = (int)(p & 255u);
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) cnt += __popcll((right ? b[t] : a[t]) & (prefix_mask(x, t) ^ (right ? 0ull : ~0ull)));
      const uint64_t base = ((uint64_t)s << BI_SHIFT) + (a[0] & 0xffffull);
      const uint64_t r = right ? base + cnt : base - cnt;
      return c == 0 ? q - r : r;
    }
    if (h.layout == QR_LAYOUT_BIRANK16X2) {
      uint64_t j = q / B16X2_B;
      j = j > last ? last : j;
      uint64_t d = q - j * B16X2_B;
      d = d > B16X2_B - 1 ? B16X2_B - 1 : d;
      const uint32_t hh = d >= 240 ? 1u : 0u;
      const int x = (int)(d - 240 * hh);
      ld_sector_na(h.lines + 4 * j + 2 * hh, a[0], a[1], a[2], a[3]);
      const uint32_t s = __ldg(h.super + (j >> BI_SB_LOG));
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) cnt += __popcll(a[t] & (prefix_mask(16 + x, t) ^ prefix_mask(136, t)));
      const uint64_t base = ((uint64_t)s << BI_SHIFT) + (a[0] & 0xffffull);
      const uint64_t r = x >= 120 ? base + cnt : base - cnt;
      return c == 0 ? q - r : r;
    }
    if (h.layout == QR_LAYOUT_BIRANK32X2) {
      uint64_t j = q / B32X2_B;
      j = j > last ? last : j;
      uint64_t d = q - j * B32X2_B;
      d = d > B32X2_B - 1 ? B32X2_B - 1 : d;
      const uint32_t hh = d >= 224 ? 1u : 0u;
      const int x = (int)(d - 224 * hh);
      ld_sector_na(h.lines + 4 * j + 2 * hh, a[0], a[1], a[2], a[3]);
      const uint64_t base = __ldg(reinterpret_cast<const unsigned long long*>(h.super) + (j >> B32X2_SB_LOG)) +
                            (a[0] & 0xffffffffull);
      uint32_t cnt = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) cnt += __popcll(a[t] & (prefix_mask(32 + x, t) ^ prefix_mask(144, t)));
      const uint64_t r = x >= 112 ? base + cnt : base - cnt;
      return c == 0 ? q - r : r;
    }
    if (h.layout == QR_LAYOUT_BIRANK64X2) {
      uint64_t j = q / 384;
      j = j > last ? last : j;
      uint64_t rr = q - j * 384;
      rr = rr > 383 ? 383 : rr;
      const uint32_t hh = rr >= 192 ? 1u : 0u;
      const int x = (int)(rr - 192 * hh);
      ld_sector_na(h.lines + 4 * j + 2 * hh, a[0], a[1], a[2], a[3]);
      const uint32_t cnt = __popcll(a[1] & (prefix_mask(x, 0) ^ ~0ull)) +
                           __popcll(a[2] & (prefix_mask(x, 1) ^ 0xffffffffull)) + __popcll(a[3] & prefix_mask(x, 2));
      const uint64_t r = x >= 96 ? a[0] + cnt : a[0] - cnt;
      return c == 0 ? q - r : r;
    }
    const uint64_t cl = 0ull - (uint64_t)(c & 1u), ch = 0ull - (uint64_t)((c >> 1) & 1u);
    if (h.layout == QR_LAYOUT_QUADRANK16) {
      uint64_t j = q / QD_B;
      j = j > last ? last : j;
      uint64_t p = 32 + q - j * QD_B;
      p = p > 255 ? 255 : p;
      const uint4* ln = h.lines + 4 * j;
      ld_sector_na(ln, a[0], a[1], a[2], a[3]);
      if (p >= 128) ld_sector_na(ln + 2, b[0], b[1], b[2], b[3]);
      const uint32_t s = __ldg(h.super + 4 * (j >> QD_SB_LOG) + (c & 3u));
      const bool right = p >= 128;
      const int x = (int)(p & 127u);
      const uint64_t* w = right ? b : a;
      const uint64_t inv = right ? 0ull : ~0ull;
      const uint32_t cnt = __popcll((w[0] ^ cl) & (w[1] ^ ch) & (prefix_mask(x, 0) ^ inv)) +
                           __popcll((w[2] ^ cl) & (w[3] ^ ch) & (prefix_mask(x, 1) ^ inv));
      const uint64_t dw = (c & 2u) ? a[1] : a[0];
      const uint64_t base = ((uint64_t)s << QD_SHIFT) + ((dw >> (16 * (c & 1u))) & 0xffffull);
      return right ? base + cnt : base - cnt;
    }
    if (h.layout == QR_LAYOUT_QUADRANK16X2) {
      uint64_t j = q / Q16X2_B;
      j = j > last ? last : j;
      uint64_t d = q - j * Q16X2_B;
      d = d > Q16X2_B - 1 ? Q16X2_B - 1 : d;
      const uint32_t hh = d >= 96 ? 1u : 0u;
      const uint32_t x = (uint32_t)d - 96u * hh;
      ld_sector_na(h.lines + 4 * j + 2 * hh, a[0], a[1], a[2], a[3]);
      const uint32_t s = __ldg(h.super + 4 * (j >> QD_SB_LOG) + (c & 3u));
      const uint64_t nl = (c & 1u) ? 0ull : ~0ull, nh = (c & 2u) ? 0ull : ~0ull;
      const uint32_t cnt = __popcll((a[1] ^ nl) & (a[2] ^ nh) & (prefix_mask((int)x, 0) ^ prefix_mask(48, 0))) +
                           __popcll((a[3] ^ nl) & ((a[3] >> 32) ^ nh) & (prefix_mask((int)x, 1) ^ prefix_mask(48, 1)) &
                                    0xffffffffull);
      const uint64_t base = ((uint64_t)s << QD_SHIFT) + ((a[0] >> (16 * (c & 3u))) & 0xffffull);
      return x >= 48 ? base + cnt : base - cnt;
    }
    // QuadRank64
    uint64_t j = q >> 7;
    j = j > last ? last : j;
    const uint64_t x = (j << 7 == (q & ~127ull)) ? (q & 127u) : 127u;
    const uint4* ln = h.lines + 4 * j;
    ld_sector_na(ln, a[0], a[1], a[2], a[3]);
    ld_sector_na(ln + 2, b[0], b[1], b[2], b[3]);
    const bool right = x >= 64;
    const int y = (int)(x & 63u);
    const uint64_t wl = right ? b[2] : b[0], wh = right ? b[3] : b[1];
    const uint32_t cnt = __popcll((wl ^ cl) & (wh ^ ch) & (prefix_mask(y, 0) ^ (right ? 0ull : ~0ull)));
    const uint64_t v = (c & 2u) ? ((c & 1u) ? a[3] : a[2]) : ((c & 1u) ? a[1] : a[0]);
    return right ? v + cnt : v - cnt;
  }
};
}  // namespace

__global__ void k_rank_chain(const qr_index h, const uint64_t* __restrict__ q, const uint8_t* __restrict__ cs,
                             uint64_t* __restrict__ out, uint64_t m, uint64_t chain_len) {
  const RankOne rank{h};
  const uint64_t chains = (m + chain_len - 1) / chain_len;
  const uint64_t np1 = h.n + 1;
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < chains; k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = 0;
    const uint64_t end = (k + 1) * chain_len < m ? (k + 1) * chain_len : m;
    for (uint64_t i = k * chain_len; i < end; ++i) {
      uint64_t qe = q[i] + r;                     // q[i] <= n and r <= n: one subtraction is the mod
      qe = qe >= np1 ? qe - np1 : qe;
      const uint32_t c = cs ? (uint32_t)cs[i] : 1u;
      r = rank(qe, c);
      out[i] = r;
    }
  }
}

cudaError_t launch_rank_chain(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                              uint64_t chain_len, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  const uint64_t chains = (m + chain_len - 1) / chain_len;
  const unsigned threads = chains < 128 ? 32u : 128u;
  uint64_t g = (chains + threads - 1) / threads;
  if (g > (uint64_t)h->sm_count * 64) g = (uint64_t)h->sm_count * 64;
  k_rank_chain<<<(unsigned)g, threads, 0, st>>>(*h, q, c, out, m, chain_len);
  return cudaGetLastError();
}

}  // namespace qr
