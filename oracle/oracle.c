/*
 * oracle.c — CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path
 * (paper_2602_04103_b200/) never links, imports or calls it, and this file shares
 * no code, header, table or constant with it.
 *
 * What it computes is the paper's *plain definitions*, not the paper's
 * algorithms: the BiRank/QuadRank layouts reach these
 * results exactly, only faster.
 *
 *   rank(q, c) := sum_{i in [0,q)} [t_i = c]          PAPER.md:61-63 (§1), :376-378 (§3)
 *   rank(q)    := rank(q, 1)  for sigma = 2
 *   FM count   := number of (overlapping) occurrences, via backward search over a
 *                 plain BWT (App. D)
 *   count_hdk  := number of text positions within Hamming distance k of the pattern
 *                 (NEXT §8(f)3), by a direct scan of every position
 *   or_scan_count / or_scan_count_bucketed := the FM count by a direct scan of every text
 *                 position (the bucketed form only skips positions whose first 8 symbols differ)
 *
 * Conventions (DESIGN.md "Readings" 1, 11, 15): bits are LE in u64 words
 * (t_i = bit i%64 of word i/64); DNA is 2-bit LE (char i = bits 2(i%32)..+1 of
 * word i/32), A=0 C=1 G=2 T=3; ranks are u64; FM counts are u32.  In this
 * oracle's BWT the sentinel '$' is the distinct byte 4 (deliberately unlike the
 * product, which stores '$' as A and corrects with its position).
 *
 * Pins (tests/test_oracle.py): brute-force sums on tiny inputs for every q,
 * rank(0)=0, rank(n)=total, increments = t_q, sum_c rank(q,c)=q, all-ones and
 * all-G special cases, naive-comparison suffix sort, brute-force substring
 * counts, SA-binary-search counts, k-mer partition identities, the worked
 * example of SPEC.md:329, and for count_hd1 / count_hdk Python brute force plus the
 * sum of exact counts over every string within distance k.  No function here is
 * "parity unpinned".
 *
 * Parallelism: an OpenMP parallel-for over independent queries/patterns only;
 * each query runs the plain definition unchanged.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

static inline uint64_t popc64(uint64_t x) { return (uint64_t)__builtin_popcountll(x); }

/* ---------------------------------------------------------------- sigma = 2 */

/* W[w] = number of 1 bits in words[0..w), w = 0..nwords.  One sequential scan. */
EXPORT void or_bits_prefix(const uint64_t* words, uint64_t nwords, uint64_t* W) {
  uint64_t acc = 0;
  for (uint64_t w = 0; w < nwords; ++w) { W[w] = acc; acc += popc64(words[w]); }
  W[nwords] = acc;
}

/* rank(q) = sum_{i<q} t_i = W[q/64] + popcount(word[q/64] & low (q%64) bits). PAPER.md:376-378 */
static inline uint64_t rank_bits_one(const uint64_t* words, const uint64_t* W, uint64_t q) {
  uint64_t w = q >> 6, r = q & 63;
  uint64_t v = W[w];
  if (r) v += popc64(words[w] & ((1ull << r) - 1ull));
  return v;
}

EXPORT void or_rank_bits(const uint64_t* words, const uint64_t* W, uint64_t n, const uint64_t* q,
                         const uint8_t* c, uint64_t m, uint64_t* out) {
  (void)n;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < (int64_t)m; ++k) {
    uint64_t r1 = rank_bits_one(words, W, q[k]);
    /* sigma = 2 with a symbol argument: rank(q,0) = q - rank(q,1) */
    out[k] = (c && c[k] == 0) ? q[k] - r1 : r1;
  }
}

/* ---------------------------------------------------------------- sigma = 4 */

static inline uint32_t dna_char(const uint64_t* text, uint64_t i) { return (uint32_t)(text[i >> 5] >> (2 * (i & 31))) & 3u; }

/* cp[4*w + c] = number of c in chars [0, 32w), w = 0..nwords.  One sequential scan, char by char. */
EXPORT void or_dna_checkpoints(const uint64_t* text, uint64_t n, uint64_t* cp) {
  uint64_t nwords = (n + 31) >> 5;
  uint64_t cnt[4] = {0, 0, 0, 0};
  for (uint64_t w = 0; w < nwords; ++w) {
    for (int c = 0; c < 4; ++c) cp[4 * w + c] = cnt[c];
    for (uint64_t i = 32 * w; i < 32 * w + 32 && i < n; ++i) cnt[dna_char(text, i)]++;
  }
  for (int c = 0; c < 4; ++c) cp[4 * nwords + c] = cnt[c];
}

/* rank(q,c) = sum_{i<q} [t_i = c] = cp[q/32][c] + scalar count over chars [32*(q/32), q). PAPER.md:61-63 */
static inline uint64_t rank_dna_one(const uint64_t* text, const uint64_t* cp, uint64_t q, uint32_t c) {
  uint64_t w = q >> 5;
  uint64_t v = cp[4 * w + c];
  for (uint64_t i = 32 * w; i < q; ++i) v += (dna_char(text, i) == c);
  return v;
}

EXPORT void or_rank_dna(const uint64_t* text, const uint64_t* cp, uint64_t n, const uint64_t* q,
                        const uint8_t* c, uint64_t m, uint64_t* out) {
  (void)n;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < (int64_t)m; ++k) out[k] = rank_dna_one(text, cp, q[k], c[k]);
}

/* rank_4(q) = (rank(q,0), rank(q,1), rank(q,2), rank(q,3)), PAPER.md:501-502 — four calls, AoS out[4k+c]. */
EXPORT void or_rank_all4_dna(const uint64_t* text, const uint64_t* cp, uint64_t n, const uint64_t* q,
                             uint64_t m, uint64_t* out4) {
  (void)n;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < (int64_t)m; ++k)
    for (uint32_t c = 0; c < 4; ++c) out4[4 * k + c] = rank_dna_one(text, cp, q[k], c);
}

/* ------------------------------------------------------- suffix array of T$ */

/* Suffix array of s[0..n) followed by the sentinel $ (smaller than every symbol).
 * Plain prefix doubling (sort suffixes by their first 2^k characters via the
 * pair (rank_k[i], rank_k[i+2^k]); stop when all ranks are distinct), with qsort
 * as the sorting primitive.  Output: sa[0..n] (n+1 entries). */
typedef struct { int64_t r1, r2; int64_t i; } sa_item;
static int sa_cmp(const void* a, const void* b) {
  const sa_item* x = (const sa_item*)a; const sa_item* y = (const sa_item*)b;
  if (x->r1 != y->r1) return x->r1 < y->r1 ? -1 : 1;
  if (x->r2 != y->r2) return x->r2 < y->r2 ? -1 : 1;
  return 0;
}
EXPORT int or_suffix_array(const uint8_t* s, uint64_t n, uint32_t* sa) {
  uint64_t N = n + 1;
  int64_t* rk = (int64_t*)malloc(N * sizeof(int64_t));
  sa_item* it = (sa_item*)malloc(N * sizeof(sa_item));
  if (!rk || !it) { free(rk); free(it); return -1; }
  for (uint64_t i = 0; i < n; ++i) rk[i] = (int64_t)s[i] + 1;   /* A..T -> 1..4 */
  rk[n] = 0;                                                     /* $ -> 0 */
  for (uint64_t k = 1;; k <<= 1) {
    for (uint64_t i = 0; i < N; ++i) {
      it[i].r1 = rk[i];
      it[i].r2 = (i + k < N) ? rk[i + k] : -1;
      it[i].i = (int64_t)i;
    }
    qsort(it, N, sizeof(sa_item), sa_cmp);
    int64_t r = 0;
    for (uint64_t j = 0; j < N; ++j) {
      if (j > 0 && sa_cmp(&it[j - 1], &it[j]) != 0) r = (int64_t)j;
      rk[it[j].i] = r;
    }
    int distinct = 1;
    for (uint64_t j = 1; j < N; ++j) if (sa_cmp(&it[j - 1], &it[j]) == 0) { distinct = 0; break; }
    if (distinct || k >= N) break;
  }
  for (uint64_t j = 0; j < N; ++j) sa[j] = (uint32_t)it[j].i;
  free(rk); free(it);
  return 0;
}

/* BWT[i] = s[sa[i]-1], or $ (= 4 here) when sa[i] = 0; spos = the row holding $. */
EXPORT void or_bwt(const uint8_t* s, uint64_t n, const uint32_t* sa, uint8_t* bwt, uint64_t* spos) {
  for (uint64_t i = 0; i <= n; ++i) {
    if (sa[i] == 0) { bwt[i] = 4; *spos = i; }
    else bwt[i] = s[sa[i] - 1];
  }
}

/* ------------------------------------------------------- FM backward search */

/* C[c] = number of characters of T$ smaller than c (with $ < A < C < G < T),
 * i.e. C[c] = 1 + #{t_i < c}; C[4] = n + 1.  cp[5*b + c] = count of c in bwt[0, 64b). */
EXPORT void or_fm_prepare(const uint8_t* bwt, uint64_t N, uint64_t* C, uint64_t* cp) {
  uint64_t cnt[5] = {0, 0, 0, 0, 0};
  uint64_t nb = N / 64 + 1;
  for (uint64_t b = 0; b < nb; ++b) {
    for (int c = 0; c < 5; ++c) cp[5 * b + c] = cnt[c];
    for (uint64_t i = 64 * b; i < 64 * b + 64 && i < N; ++i) cnt[bwt[i]]++;
  }
  C[0] = 1;                                   /* only $ is smaller than A */
  for (int c = 1; c < 4; ++c) C[c] = C[c - 1] + cnt[c - 1];
  C[4] = N;
}

/* Occ(c, x) = number of c in bwt[0, x). */
static inline uint64_t occ(const uint8_t* bwt, const uint64_t* cp, uint64_t x, uint32_t c) {
  uint64_t b = x >> 6;
  uint64_t v = cp[5 * b + c];
  for (uint64_t i = 64 * b; i < x; ++i) v += (bwt[i] == c);
  return v;
}

/* Backward search (FM-index, "rank queries and LF-mapping"):
 *   [lo, hi) = [0, n+1);  for k = len-1 .. 0:  c = P[k];
 *   lo = C[c] + Occ(c, lo);  hi = C[c] + Occ(c, hi);  stop when lo >= hi.
 * count = hi - lo (0 when empty).  No k-mer table.  steps (optional) = number of
 * backward steps executed.  Patterns: symbols 0..3, pattern k at off[k], length len[k]. */
EXPORT void or_fm_count(const uint8_t* bwt, const uint64_t* cp, const uint64_t* C, uint64_t N,
                        const uint8_t* pat, const uint64_t* off, const uint32_t* len, uint64_t m,
                        uint32_t* out, uint32_t* steps) {
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t k = 0; k < (int64_t)m; ++k) {
    const uint8_t* P = pat + off[k];
    uint64_t lo = 0, hi = N;
    uint32_t st = 0;
    for (int64_t j = (int64_t)len[k] - 1; j >= 0 && lo < hi; --j) {
      uint32_t c = P[j];
      lo = C[c] + occ(bwt, cp, lo, c);
      hi = C[c] + occ(bwt, cp, hi, c);
      ++st;
    }
    out[k] = (uint32_t)(lo < hi ? hi - lo : 0);
    if (steps) steps[k] = st;
  }
}

/* Instrumented backward search (SURVEY.md §8(c) "Instrumented mode"): for each
 * pattern, after skipping the first `skip` steps (the ones a k-mer table seeds),
 * report the number of steps and the number of distinct lines of `block` rows
 * touched ((lo/block != hi/block) ? 2 : 1 per step).  Measurement only. */
EXPORT void or_fm_work(const uint8_t* bwt, const uint64_t* cp, const uint64_t* C, uint64_t N,
                       const uint8_t* pat, const uint64_t* off, const uint32_t* len, uint64_t m,
                       uint32_t skip, uint64_t block, uint64_t* total_steps, uint64_t* total_lines) {
  uint64_t ts = 0, tl = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : ts, tl)
  for (int64_t k = 0; k < (int64_t)m; ++k) {
    const uint8_t* P = pat + off[k];
    uint64_t lo = 0, hi = N;
    uint32_t st = 0;
    uint32_t sk = len[k] >= skip ? skip : 0;   /* a k-mer table seeds only patterns of >= skip symbols */
    for (int64_t j = (int64_t)len[k] - 1; j >= 0 && lo < hi; --j) {
      uint32_t c = P[j];
      if (st >= sk) { ts += 1; tl += (lo / block != hi / block) ? 2 : 1; }
      lo = C[c] + occ(bwt, cp, lo, c);
      hi = C[c] + occ(bwt, cp, hi, c);
      ++st;
    }
  }
  *total_steps = ts; *total_lines = tl;
}

/* Second, independent counter: binary search in the suffix array for the block
 * of suffixes that start with P (suffix i of T$ compares as s[i..n) then $). */
static int cmp_suffix_pattern(const uint8_t* s, uint64_t n, uint64_t i, const uint8_t* P, uint32_t L) {
  for (uint32_t j = 0; j < L; ++j) {
    if (i + j >= n) return -1;            /* suffix hits $ first: smaller */
    if (s[i + j] != P[j]) return s[i + j] < P[j] ? -1 : 1;
  }
  return 0;                               /* P is a prefix of the suffix */
}
EXPORT void or_sa_count(const uint8_t* s, uint64_t n, const uint32_t* sa, const uint8_t* pat,
                        const uint64_t* off, const uint32_t* len, uint64_t m, uint32_t* out) {
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t k = 0; k < (int64_t)m; ++k) {
    const uint8_t* P = pat + off[k];
    uint32_t L = len[k];
    uint64_t a = 0, b = n + 1;                       /* first suffix >= P */
    while (a < b) { uint64_t mid = (a + b) / 2; if (cmp_suffix_pattern(s, n, sa[mid], P, L) < 0) a = mid + 1; else b = mid; }
    uint64_t lo = a;
    b = n + 1;                                        /* first suffix > P (not prefixed by P) */
    while (a < b) { uint64_t mid = (a + b) / 2; if (cmp_suffix_pattern(s, n, sa[mid], P, L) <= 0) a = mid + 1; else b = mid; }
    out[k] = (uint32_t)(a - lo);
  }
}

/* Third counter: direct scan of every text position (overlapping occurrences).
 * An empty pattern occurs at every one of the n+1 positions. */
EXPORT void or_scan_count(const uint8_t* s, uint64_t n, const uint8_t* pat, const uint64_t* off,
                          const uint32_t* len, uint64_t m, uint32_t* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < (int64_t)m; ++k) {
    const uint8_t* P = pat + off[k];
    uint32_t L = len[k];
    uint64_t cnt = 0;
    if (L == 0) cnt = n + 1;
    else if (L <= n)
      for (uint64_t i = 0; i + L <= n; ++i) {
        uint32_t j = 0;
        while (j < L && s[i + j] == P[j]) ++j;
        cnt += (j == L);
      }
    out[k] = (uint32_t)cnt;
  }
}

/* The same count as or_scan_count — the number of (overlapping) text positions where the whole
 * pattern matches — for large batches on large texts: the patterns of >= 8
 * symbols are grouped by their first 8 symbols, and each text position is compared in full only
 * with the patterns whose first 8 symbols equal the text's there (a pattern whose first 8
 * symbols differ cannot occur at that position); shorter patterns take or_scan_count.  Loop order
 * and filtering only: every count is still a direct comparison at every position.  Pinned against
 * or_scan_count and Python brute force (tests/test_oracle.py). */
EXPORT void or_scan_count_bucketed(const uint8_t* s, uint64_t n, const uint8_t* pat, const uint64_t* off,
                                   const uint32_t* len, uint64_t m, uint32_t* out) {
  const uint32_t NB = 1u << 16;                      /* 8 symbols, 2 bits each */
  uint32_t* head = (uint32_t*)calloc(NB + 1, sizeof(uint32_t));
  uint32_t* list = (uint32_t*)malloc((m ? m : 1) * sizeof(uint32_t));
  uint64_t* cnt = (uint64_t*)calloc(m ? m : 1, sizeof(uint64_t));
  uint64_t k;
  for (k = 0; k < m; ++k) {                          /* counting sort of the long patterns by key */
    if (len[k] < 8) continue;
    uint32_t key = 0;
    for (int j = 0; j < 8; ++j) key = (key << 2) | (pat[off[k] + j] & 3u);
    head[key + 1]++;
  }
  for (uint32_t b = 0; b < NB; ++b) head[b + 1] += head[b];
  uint32_t* fill = (uint32_t*)malloc(NB * sizeof(uint32_t));
  memcpy(fill, head, NB * sizeof(uint32_t));
  for (k = 0; k < m; ++k) {
    if (len[k] < 8) continue;
    uint32_t key = 0;
    for (int j = 0; j < 8; ++j) key = (key << 2) | (pat[off[k] + j] & 3u);
    list[fill[key]++] = (uint32_t)k;
  }
  free(fill);
  if (n >= 8) {
#pragma omp parallel
    {
      uint64_t* loc = (uint64_t*)calloc(m ? m : 1, sizeof(uint64_t));
#pragma omp for schedule(static)
      for (int64_t i = 0; i <= (int64_t)n - 8; ++i) {
        uint32_t key = 0;
        for (int j = 0; j < 8; ++j) key = (key << 2) | s[i + j];
        for (uint32_t t = head[key]; t < head[key + 1]; ++t) {
          const uint32_t q = list[t];
          const uint32_t L = len[q];
          if ((uint64_t)i + L > n) continue;
          if (memcmp(s + i, pat + off[q], L) == 0) loc[q]++;
        }
      }
#pragma omp critical
      for (uint64_t q = 0; q < m; ++q) cnt[q] += loc[q];
      free(loc);
    }
  }
  for (k = 0; k < m; ++k) {
    if (len[k] >= 8) { out[k] = (uint32_t)cnt[k]; continue; }
    or_scan_count(s, n, pat, off + k, len + k, 1, out + k);   /* short patterns: the plain scan */
  }
  free(head); free(list); free(cnt);
}

/* Approximate occurrences (NEXT §8(f)3; the paper's motivation for rank_4):
 * the number of text positions i in [0, n-L] where s[i..i+L) differs from P in at most one
 * symbol (Hamming distance <= 1).  Direct scan of every position.  L = 0 counts n+1. */
EXPORT void or_scan_count_hd1(const uint8_t* s, uint64_t n, const uint8_t* pat, const uint64_t* off,
                              const uint32_t* len, uint64_t m, uint32_t* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t k = 0; k < (int64_t)m; ++k) {
    const uint8_t* P = pat + off[k];
    uint32_t L = len[k];
    uint64_t cnt = 0;
    if (L == 0) cnt = n + 1;
    else if (L <= n)
      for (uint64_t i = 0; i + L <= n; ++i) {
        uint32_t mism = 0;
        for (uint32_t j = 0; j < L && mism <= 1; ++j) mism += (s[i + j] != P[j]);
        cnt += (mism <= 1);
      }
    out[k] = (uint32_t)cnt;
  }
}

/* Approximate occurrences with up to k substitutions (NEXT §8(f)3 widened beyond one
 * substitution): the number of text positions i in [0, n-L] where s[i..i+L)
 * differs from P in at most k symbols (Hamming distance <= k).  Direct scan of every position;
 * L = 0 counts n+1. */
EXPORT void or_scan_count_hdk(const uint8_t* s, uint64_t n, const uint8_t* pat, const uint64_t* off,
                              const uint32_t* len, uint64_t m, uint32_t k, uint32_t* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < (int64_t)m; ++t) {
    const uint8_t* P = pat + off[t];
    uint32_t L = len[t];
    uint64_t cnt = 0;
    if (L == 0) cnt = n + 1;
    else if (L <= n)
      for (uint64_t i = 0; i + L <= n; ++i) {
        uint32_t mism = 0;
        for (uint32_t j = 0; j < L && mism <= k; ++j) mism += (s[i + j] != P[j]);
        cnt += (mism <= k);
      }
    out[t] = (uint32_t)cnt;
  }
}

EXPORT int or_threads(void) { return omp_get_max_threads(); }
/* Threads of the parallel-for over queries (a launcher such as torchrun may have set
 * OMP_NUM_THREADS=1 for every rank; the host baseline runs on rank 0 alone). */
EXPORT void or_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
