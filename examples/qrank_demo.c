/*
 * qrank_demo.c — using libqrank.so from plain C (C99), no Python, no CUDA headers.
 *
 * Builds a BiRank16 index over a bit vector, a QuadRank16 index and a QuadFm index over a DNA
 * text, all from HOST buffers, and queries them from host buffers (the library's staged
 * host<->device path).  Every answer is checked against a naive loop written here, so the
 * program doubles as a smoke test of the C boundary on a GPU box:
 *
 *     make examples/qrank_demo && ./examples/qrank_demo      (exit 0 and "qrank_demo OK")
 *
 * The checks are the plain definitions: rank(q) = #{i < q : t_i = 1},
 * rank(q, c) = #{i < q : t_i = c}, and occurrence counts by scanning every text position.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "qrank.h"

static uint64_t rng_state = 0x9e3779b97f4a7c15ull;
static uint64_t next_u64(void) {                   /* xorshift64*, demo data only */
  rng_state ^= rng_state >> 12;
  rng_state ^= rng_state << 25;
  rng_state ^= rng_state >> 27;
  return rng_state * 0x2545f4914f6cdd1dull;
}

#define CHECK(call)                                                                     \
  do {                                                                                  \
    qr_status st_ = (call);                                                             \
    if (st_ != QR_OK) {                                                                 \
      fprintf(stderr, "%s:%d: %s -> status %d: %s\n", __FILE__, __LINE__, #call, st_, \
              qr_last_error());                                                         \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)

static unsigned sym_at(const uint64_t* t, uint64_t i) { return (unsigned)(t[i >> 5] >> (2 * (i & 31))) & 3u; }

int main(void) {
  printf("%s\n", qr_version());

  /* ---- BiRank16: n bits, m random queries in [0, n] ---- */
  const uint64_t n = 1000003, m = 4096;
  uint64_t* bits = calloc((n + 63) / 64, 8);
  for (uint64_t w = 0; w < (n + 63) / 64; ++w) bits[w] = next_u64();
  if (n % 64) bits[n / 64] &= (1ull << (n % 64)) - 1;
  qr_index* bi = NULL;
  CHECK(qr_birank_build(bits, n, 0, NULL, &bi));
  uint64_t* q = malloc(m * 8);
  uint64_t* out = malloc(m * 8);
  for (uint64_t i = 0; i < m; ++i) q[i] = next_u64() % (n + 1);
  q[0] = 0; q[1] = n;
  CHECK(qr_rank(bi, q, NULL, out, m, NULL));
  CHECK(qr_sync(NULL));
  for (uint64_t i = 0; i < m; ++i) {
    uint64_t r = 0;
    for (uint64_t b = 0; b < q[i]; ++b) r += (bits[b >> 6] >> (b & 63)) & 1u;
    if (r != out[i]) { fprintf(stderr, "BiRank rank(%llu) = %llu, expected %llu\n",
                                (unsigned long long)q[i], (unsigned long long)out[i], (unsigned long long)r); return 1; }
  }
  qr_free(bi);

  /* ---- QuadRank16: n4 DNA symbols (2 bits each), rank_4 on host buffers ---- */
  const uint64_t n4 = 200001, m4 = 2048;
  uint64_t* txt = calloc((n4 + 31) / 32 + 1, 8);
  for (uint64_t w = 0; w < (n4 + 31) / 32; ++w) txt[w] = next_u64();
  if (n4 % 32) txt[n4 / 32] &= (1ull << (2 * (n4 % 32))) - 1;
  qr_index* qd = NULL;
  CHECK(qr_quadrank_build(txt, n4, 0, NULL, &qd));
  uint64_t* out4 = malloc(m4 * 32);
  for (uint64_t i = 0; i < m4; ++i) q[i] = next_u64() % (n4 + 1);
  CHECK(qr_rank_all4(qd, q, out4, m4, NULL));
  CHECK(qr_sync(NULL));
  for (uint64_t i = 0; i < m4; ++i) {
    uint64_t r[4] = {0, 0, 0, 0};
    for (uint64_t k = 0; k < q[i]; ++k) r[sym_at(txt, k)]++;
    for (int c = 0; c < 4; ++c)
      if (r[c] != out4[4 * i + c]) { fprintf(stderr, "QuadRank rank_4 mismatch at q=%llu c=%d\n",
                                              (unsigned long long)q[i], c); return 1; }
  }
  qr_free(qd);

  /* ---- QuadFm: count m patterns of length L (half are substrings of the text) ---- */
  const uint32_t L = 12;
  const uint64_t mp = 256;
  qr_fm* fm = NULL;
  CHECK(qr_fm_build(txt, n4, NULL, 0, NULL, &fm));
  uint8_t* pats = malloc(mp * L + 8);
  uint32_t* cnt = malloc(mp * 4);
  for (uint64_t i = 0; i < mp; ++i) {
    uint64_t a = next_u64() % (n4 - L + 1);
    for (uint32_t k = 0; k < L; ++k) pats[i * L + k] = (i & 1) ? (uint8_t)(next_u64() & 3u) : (uint8_t)sym_at(txt, a + k);
  }
  CHECK(qr_fm_count(fm, pats, NULL, L, cnt, mp, NULL));
  CHECK(qr_sync(NULL));
  for (uint64_t i = 0; i < mp; ++i) {
    uint32_t r = 0;
    for (uint64_t a = 0; a + L <= n4; ++a) {
      uint32_t k = 0;
      while (k < L && sym_at(txt, a + k) == pats[i * L + k]) ++k;
      r += (k == L);
    }
    if (r != cnt[i] || (!(i & 1) && r == 0)) { fprintf(stderr, "QuadFm count mismatch for pattern %llu\n",
                                                       (unsigned long long)i); return 1; }
  }
  qr_fm_free(fm);

  /* ---- errors are status codes with a message, never crashes ---- */
  if (qr_rank_all4(NULL, q, out4, 1, NULL) != QR_EINVAL) { fprintf(stderr, "expected QR_EINVAL\n"); return 1; }

  free(bits); free(q); free(out); free(txt); free(out4); free(pats); free(cnt);
  printf("qrank_demo OK\n");
  return 0;
}
