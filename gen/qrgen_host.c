/*
 * qrgen_host.c — host fill functions of the seeded generators (gen/qrgen.h).
 * Harness only: no rank / layout / FM arithmetic here.
 * Threads: OpenMP over independent output words; output is a pure function of
 * (seed, index), so it does not depend on the thread count.
 */
#include "qrgen.h"
#include <omp.h>
#include <stddef.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* n bits, p = thr/2^64, or word mode when word_mode != 0 (p = 0.5). Tail bits >= n are 0. */
EXPORT void qrgen_bits_host(uint64_t seed, uint64_t n, int word_mode, uint64_t thr, uint64_t* words) {
  int64_t nw = (int64_t)((n + 63) >> 6);
#pragma omp parallel for schedule(static)
  for (int64_t w = 0; w < nw; ++w) {
    uint64_t x = word_mode ? qrg_word(seed, QRG_TAG_BITS, (uint64_t)w) : qrg_bern_word(seed, (uint64_t)w, thr);
    uint64_t lo = (uint64_t)w << 6;
    if (lo + 64 > n) x &= (n - lo == 64) ? ~0ull : ((1ull << (n - lo)) - 1ull);
    words[w] = x;
  }
}

/* n DNA chars, 2-bit LE packed; kind 0 = iid, kind 1 = block-repeat (config 5). Tail chars are 0. */
EXPORT void qrgen_dna_host(uint64_t seed, uint64_t n, int kind, uint64_t* words) {
  int64_t nw = (int64_t)((n + 31) >> 5);
#pragma omp parallel for schedule(static)
  for (int64_t w = 0; w < nw; ++w) {
    uint64_t x = 0;
    uint64_t lo = (uint64_t)w << 5;
    if (kind == 0) {
      x = qrg_word(seed, QRG_TAG_DNA, (uint64_t)w);
      if (lo + 32 > n) x &= (n - lo == 32) ? ~0ull : ((1ull << (2 * (n - lo))) - 1ull);
    } else {
      for (uint64_t k = 0; k < 32 && lo + k < n; ++k) x |= (uint64_t)qrg_rep_char(seed, lo + k) << (2 * k);
    }
    words[w] = x;
  }
}

/* queries i in [i0, i0+m): q u64 in [0,n]; c (optional) u8 in 0..3 */
EXPORT void qrgen_queries_host(uint64_t seed, uint64_t n, uint64_t i0, uint64_t m, uint64_t* q, uint8_t* c) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < (int64_t)m; ++k) {
    if (q) q[k] = qrg_query(seed, i0 + (uint64_t)k, n);
    if (c) c[k] = qrg_qsym(seed, i0 + (uint64_t)k);
  }
}

/* m patterns i in [i0, i0+m) of fixed length len, concatenated */
EXPORT void qrgen_patterns_host(uint64_t seed, int kind, uint64_t i0, uint64_t m, uint32_t len,
                                const uint64_t* text2b, uint64_t n, uint8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < (int64_t)m; ++k)
    qrg_pattern(seed, kind, i0 + (uint64_t)k, len, text2b, n, out + (size_t)k * len);
}

/* unpack 2-bit text into one byte per symbol */
EXPORT void qrgen_unpack_dna_host(const uint64_t* words, uint64_t n, uint8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = (uint8_t)qrg_text_char(words, (uint64_t)i);
}

EXPORT int qrgen_host_threads(void) { return omp_get_max_threads(); }
