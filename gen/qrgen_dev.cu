/*
 * qrgen_dev.cu — device fill kernels of the seeded generators (gen/qrgen.h).
 * Harness only.  Bit-identical to qrgen_host.c.
 * Every entry point is stream-ordered on `stream` (a cudaStream_t as void*).
 */
#include "qrgen.h"
#include <cuda_runtime.h>

#define EXPORT extern "C" __attribute__((visibility("default")))

static unsigned grid_for(uint64_t items, unsigned threads) {
  uint64_t g = (items + threads - 1) / threads;
  if (g > 148ull * 64ull) g = 148ull * 64ull;   /* grid-stride beyond 64 waves of CTAs */
  return g ? (unsigned)g : 1u;
}

__global__ void k_bits(uint64_t seed, uint64_t n, int word_mode, uint64_t thr, uint64_t* words) {
  uint64_t nw = (n + 63) >> 6;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = word_mode ? qrg_word(seed, QRG_TAG_BITS, w) : qrg_bern_word(seed, w, thr);
    uint64_t lo = w << 6;
    if (lo + 64 > n) x &= (n - lo == 64) ? ~0ull : ((1ull << (n - lo)) - 1ull);
    words[w] = x;
  }
}

__global__ void k_dna(uint64_t seed, uint64_t n, int kind, uint64_t* words) {
  uint64_t nw = (n + 31) >> 5;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = 0, lo = w << 5;
    if (kind == 0) {
      x = qrg_word(seed, QRG_TAG_DNA, w);
      if (lo + 32 > n) x &= (n - lo == 32) ? ~0ull : ((1ull << (2 * (n - lo))) - 1ull);
    } else {
      for (uint64_t k = 0; k < 32 && lo + k < n; ++k) x |= (uint64_t)qrg_rep_char(seed, lo + k) << (2 * k);
    }
    words[w] = x;
  }
}

__global__ void k_queries(uint64_t seed, uint64_t n, uint64_t i0, uint64_t m, uint64_t* q, uint8_t* c) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
    if (q) q[k] = qrg_query(seed, i0 + k, n);
    if (c) c[k] = qrg_qsym(seed, i0 + k);
  }
}

__global__ void k_patterns(uint64_t seed, int kind, uint64_t i0, uint64_t m, uint32_t len,
                           const uint64_t* text2b, uint64_t n, uint8_t* out) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x)
    qrg_pattern(seed, kind, i0 + k, len, text2b, n, out + k * len);
}

EXPORT int qrgen_bits_dev(uint64_t seed, uint64_t n, int word_mode, uint64_t thr, uint64_t* words, void* stream) {
  k_bits<<<grid_for((n + 63) >> 6, 256), 256, 0, (cudaStream_t)stream>>>(seed, n, word_mode, thr, words);
  return (int)cudaGetLastError();
}
EXPORT int qrgen_dna_dev(uint64_t seed, uint64_t n, int kind, uint64_t* words, void* stream) {
  k_dna<<<grid_for((n + 31) >> 5, 256), 256, 0, (cudaStream_t)stream>>>(seed, n, kind, words);
  return (int)cudaGetLastError();
}
EXPORT int qrgen_queries_dev(uint64_t seed, uint64_t n, uint64_t i0, uint64_t m, uint64_t* q, uint8_t* c, void* stream) {
  k_queries<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(seed, n, i0, m, q, c);
  return (int)cudaGetLastError();
}
EXPORT int qrgen_patterns_dev(uint64_t seed, int kind, uint64_t i0, uint64_t m, uint32_t len,
                              const uint64_t* text2b, uint64_t n, uint8_t* out, void* stream) {
  k_patterns<<<grid_for(m, 128), 128, 0, (cudaStream_t)stream>>>(seed, kind, i0, m, len, text2b, n, out);
  return (int)cudaGetLastError();
}
