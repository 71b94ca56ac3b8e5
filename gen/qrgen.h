/*
 * qrgen.h — seeded, counter-based synthetic-input generators (harness step a9,
 * SURVEY.md §8(a)/§8(d) "Generators (G0)").
 *
 * This module is the ONLY code shared by the CUDA product path
 * (paper_2602_04103_b200/) and the CPU oracle's tests (oracle/, tests/).  It holds
 * none of the method's arithmetic: no rank, no layout, no BWT.  It only
 * produces texts, query positions, query symbols and FM patterns, each value a
 * pure function of (seed, stream tag, index), so the host (qrgen_host.c) and the
 * device (qrgen_dev.cu) produce bit-identical streams without exchanging data.
 *
 * Generator: h(seed, tag, i) = splitmix64 finaliser of
 *            (seed ^ tag*0xD1B54A32D192ED03) + (i+1)*0x9E3779B97F4A7C15.
 * Uniform in [0, N): mulhi64(h, N).  Bernoulli(p): h < floor(p*2^64).
 *
 * Workload recipes:
 *   bits, p = 0.5   : word w = h(seed, BITS, w)            (LE: t_i = bit i%64 of word i/64)
 *   bits, other p   : bit i = [h(seed, BITS, i) < p*2^64]
 *   DNA iid         : word w = h(seed, DNA, w)             (char i = bits 2(i%32)..+1 of word i/32)
 *   DNA block-repeat: blocks of QRG_BLOCK symbols; block b>0 is, with prob. 0.3, a copy of
 *                     block mulhi(h(seed,SRC,b), b) with per-position Bernoulli(0.01)
 *                     substitutions by one of the 3 other symbols; else iid h(seed,DNA,.)
 *   queries         : q_i = mulhi(h(seed, Q, i), n+1) in [0, n];   c_i = h(seed, C, i) & 3
 *   patterns        : see qrg_pattern_* below.
 */
#ifndef QRGEN_H
#define QRGEN_H
#include <stdint.h>

#ifdef __CUDACC__
#define QRG_HD __host__ __device__ __forceinline__
#else
#define QRG_HD static inline
#endif

/* stream tags */
#define QRG_TAG_BITS   1u
#define QRG_TAG_DNA    2u
#define QRG_TAG_Q      3u
#define QRG_TAG_C      4u
#define QRG_TAG_BLK    5u
#define QRG_TAG_SRC    6u
#define QRG_TAG_MUT    7u
#define QRG_TAG_MSYM   8u
#define QRG_TAG_PPOS   9u
#define QRG_TAG_PCHR  10u
#define QRG_TAG_PKIND 11u
#define QRG_TAG_PSUB  12u
#define QRG_TAG_RMUT  13u
#define QRG_TAG_RSYM  14u
#define QRG_TAG_RSTR  15u

#define QRG_BLOCK 10000ull          /* config 5 block length (BASELINE.json configs[4]) */
#define QRG_P_COPY  0x4CCCCCCCCCCCCCCDull   /* ceil(0.3 * 2^64)  */
#define QRG_P_MUT   0x028F5C28F5C28F5Cull   /* floor(0.01 * 2^64) */

QRG_HD uint64_t qrg_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
QRG_HD uint64_t qrg_hash(uint64_t seed, uint64_t tag, uint64_t i) {
  return qrg_mix((seed ^ (tag * 0xD1B54A32D192ED03ull)) + (i + 1ull) * 0x9E3779B97F4A7C15ull);
}
QRG_HD uint64_t qrg_mulhi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * (unsigned __int128)b) >> 64);
#endif
}
/* uniform in [0, N) */
QRG_HD uint64_t qrg_below(uint64_t seed, uint64_t tag, uint64_t i, uint64_t N) {
  return qrg_mulhi(qrg_hash(seed, tag, i), N);
}

/* one 64-bit word (32 DNA chars or 64 bits) of the iid streams */
QRG_HD uint64_t qrg_word(uint64_t seed, uint64_t tag, uint64_t w) { return qrg_hash(seed, tag, w); }

/* 64 Bernoulli(thr/2^64) bits, bit i of word w = [h(seed,BITS,64w+i) < thr] */
QRG_HD uint64_t qrg_bern_word(uint64_t seed, uint64_t w, uint64_t thr) {
  uint64_t x = 0;
  for (int b = 0; b < 64; ++b)
    x |= (uint64_t)(qrg_hash(seed, QRG_TAG_BITS, 64ull * w + (uint64_t)b) < thr) << b;
  return x;
}

/* iid DNA character at global position i */
QRG_HD uint32_t qrg_dna_char(uint64_t seed, uint64_t i) {
  return (uint32_t)(qrg_hash(seed, QRG_TAG_DNA, i >> 5) >> (2 * (i & 31))) & 3u;
}

/* block-repeat DNA character at global position i (config 5) */
QRG_HD uint32_t qrg_rep_char(uint64_t seed, uint64_t i) {
  uint64_t b = i / QRG_BLOCK, k = i - b * QRG_BLOCK;
  /* Follow the copy chain back to an iid block, applying each link's
   * substitution at this offset on the way back (outermost link wins,
   * so we record mutations in chain order and apply them innermost-first). */
  uint64_t chain[64];
  int depth = 0;
  while (b > 0 && qrg_hash(seed, QRG_TAG_BLK, b) < QRG_P_COPY && depth < 64) {
    chain[depth++] = b;
    b = qrg_below(seed, QRG_TAG_SRC, b, b);
  }
  uint32_t c = qrg_dna_char(seed, b * QRG_BLOCK + k);
  for (int d = depth - 1; d >= 0; --d) {
    uint64_t pos = chain[d] * QRG_BLOCK + k;
    if (qrg_hash(seed, QRG_TAG_MUT, pos) < QRG_P_MUT)
      c = (c + 1u + (uint32_t)qrg_below(seed, QRG_TAG_MSYM, pos, 3)) & 3u;
  }
  return c;
}

/* query position in [0, n] and symbol */
QRG_HD uint64_t qrg_query(uint64_t seed, uint64_t i, uint64_t n) { return qrg_below(seed, QRG_TAG_Q, i, n + 1ull); }
QRG_HD uint8_t qrg_qsym(uint64_t seed, uint64_t i) { return (uint8_t)(qrg_hash(seed, QRG_TAG_C, i) & 3u); }

/* 2-bit character k of a packed text */
QRG_HD uint32_t qrg_text_char(const uint64_t* text2b, uint64_t k) {
  return (uint32_t)(text2b[k >> 5] >> (2 * (k & 31))) & 3u;
}

/*
 * FM patterns.
 * kind 0 ("config 4"): pattern i of length len; even i = exact substring of the
 *   text at mulhi(h(PPOS,i), n-len+1); odd i = len iid symbols h(PCHR, i*len+k)&3.
 * kind 1 ("config 5"): substring at mulhi(h(PPOS,i), n-len+1) with s = mulhi(h(PKIND,i),3)
 *   substitutions at distinct positions (rejection on the PSUB stream), each
 *   replaced by one of the 3 other symbols uniformly.
 * kind 2 ("reads", the paper's FM workload shape): substring at
 *   mulhi(h(PPOS,i), n-len+1), each position independently substituted with probability 0.01
 *   (RMUT stream) by one of the 3 other symbols (RSYM), then reverse-complemented when
 *   h(RSTR,i) is odd (reads come from either strand).
 * Writes len symbols (0..3, one byte each) to out.
 */
QRG_HD void qrg_pattern(uint64_t seed, int kind, uint64_t i, uint32_t len,
                        const uint64_t* text2b, uint64_t n, uint8_t* out) {
  uint64_t span = (n >= len) ? (n - len + 1ull) : 1ull;
  if (kind == 0 && (i & 1ull)) {
    for (uint32_t k = 0; k < len; ++k)
      out[k] = (uint8_t)(qrg_hash(seed, QRG_TAG_PCHR, i * (uint64_t)len + k) & 3u);
    return;
  }
  uint64_t pos = qrg_below(seed, QRG_TAG_PPOS, i, span);
  for (uint32_t k = 0; k < len; ++k)
    out[k] = (pos + k < n) ? (uint8_t)qrg_text_char(text2b, pos + k) : (uint8_t)0;
  if (kind == 2) {
    for (uint32_t k = 0; k < len; ++k)
      if (qrg_hash(seed, QRG_TAG_RMUT, i * (uint64_t)len + k) < QRG_P_MUT)
        out[k] = (uint8_t)((out[k] + 1u + (uint32_t)qrg_below(seed, QRG_TAG_RSYM, i * (uint64_t)len + k, 3)) & 3u);
    if (qrg_hash(seed, QRG_TAG_RSTR, i) & 1u)
      for (uint32_t a = 0, b = len - 1; a <= b && b < len; ++a, --b) {
        uint8_t x = (uint8_t)(3u - out[a]), y = (uint8_t)(3u - out[b]);
        out[a] = y;
        out[b] = x;
        if (b == 0) break;
      }
    return;
  }
  if (kind == 1 && len > 0) {
    uint32_t s = (uint32_t)qrg_below(seed, QRG_TAG_PKIND, i, 3);
    uint32_t used[2] = {0xffffffffu, 0xffffffffu};
    uint64_t ctr = 0;
    for (uint32_t t = 0; t < s && t < len; ++t) {
      uint32_t p;
      do {
        p = (uint32_t)qrg_below(seed, QRG_TAG_PSUB, i * 64ull + ctr, len);
        ++ctr;
      } while (p == used[0] || p == used[1]);
      used[t] = p;
      uint32_t r = (uint32_t)qrg_below(seed, QRG_TAG_PSUB, i * 64ull + 32ull + t, 3);
      out[p] = (uint8_t)((out[p] + 1u + r) & 3u);
    }
  }
}

#endif
