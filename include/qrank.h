/*
 * qrank.h — C ABI of the B200-native rank / QuadFm library
 * (libqrank.so; arXiv 2602.04103 "BiRank / QuadRank / QuadFm").
 *
 * Citations: PAPER.md line numbers with their section; SPEC.md lines as S:n.
 *
 * Definitions the calls compute (§1, lines 55-66):
 *     rank(q, c) := #{ i in [0, q) : t_i = c },   0 <= q <= n;   rank(q) := rank(q, 1) for sigma = 2.
 *
 * Text encodings (reading R1):
 *   bits   : n bits in u64 words, little-endian: t_i = bit (i % 64) of word i / 64.
 *   DNA    : n symbols, 2 bits each, little-endian: t_i = bits 2(i%32)..2(i%32)+1 of word i/32;
 *            A = 0, C = 1, G = 2, T = 3.
 * Bits/symbols at positions >= n in the last word are ignored (the builder masks them).
 *
 * Ownership and memory spaces:
 *   - A handle owns the device memory of its layout and frees it in qr_free / qr_fm_free.
 *     Handles are immutable after build and may be used concurrently from any number of
 *     host threads and CUDA streams.
 *   - Build inputs may be host or device pointers (detected with cudaPointerGetAttributes);
 *     the library copies what it needs and never retains the caller's pointer.
 *   - Query arrays (q, c, out, patterns, lengths) are either ALL device pointers on the
 *     handle's device (fast path: one kernel launch, fully asynchronous on `stream`), or ALL
 *     host pointers (staged path: chunked host->device copy, kernel, device->host copy,
 *     pipelined over internal streams, 3 by default, knob stage_slots; `stream` is made to
 *     wait for the whole pipeline; pinned host memory gives overlap, pageable memory works
 *     but serialises).
 *     Mixed spaces are QR_EINVAL.
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *
 * Errors: every call returns a qr_status; no exception crosses the ABI.  On failure,
 * qr_last_error() returns a thread-local message.  Asynchronous kernel faults surface
 * on the next call or on qr_sync().
 */
#ifndef QRANK_H
#define QRANK_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t qr_status;
#define QR_OK        0
#define QR_EINVAL    1  /* null pointer, wrong sigma, bad enum, mixed host/device pointers    */
#define QR_ECAPACITY 2  /* n >= 2^43 (sigma=2), n >= 2^45 (sigma=4,          */
                        /* PAPER.md:514-515), or n+1 >= 2^32 for QuadFm (u32 counts)          */
#define QR_ENOMEM    3  /* device or host allocation failed                                   */
#define QR_ECUDA     4  /* a CUDA runtime call or kernel launch failed                        */
#define QR_ERANGE    5  /* opt-in range check (qr_set_tuning("check_range", 1)): some q > n     */
                        /* (PAPER.md:57 defines rank for 0 <= q <= n); the call still ran —     */
                        /* memory-safe, those outputs unspecified — and qr_last_error() says   */
                        /* how many queries were out of range.  The checked call synchronises  */
                        /* its stream, so it cannot be captured in a CUDA graph.               */

typedef struct qr_index qr_index;   /* a rank layout (QR_LAYOUT_*)                             */

/* Rank layouts.  BIRANK16 / QUADRANK16 are the paper's headline structures (§3, §4); the others
 * are variants the paper evaluates (NEXT §8(f)4): BiRank64x2 (33.3%: each 32-B
 * sector = u64 rank to the sector's middle + 192 data bits, so a query reads one sector and no
 * superblock word), QuadRank64 (100%: four u64 ranks to the middle of 128
 * characters in sector 0, the characters as two transposed negated plane pairs in sector 1) and
 * BiRank16x2 (6.72%: each 32-B sector = u16 delta to its middle + 240 data
 * bits, superblocks as BiRank16, so a query reads one sector and the superblock word), and
 * QuadRank16x2 (B200 sector-local σ=4 variant, 33.3%: each 32-B sector = four u16 deltas to its
 * middle + 96 characters as bit planes, superblocks as QuadRank16; rank and rank_4 read one
 * sector) and BiRank32x2 (14.3%: each 32-B sector = u32 delta to its middle +
 * 224 data bits, a u64 L1 entry per 2^23 lines — small enough to sit in every CTA's shared
 * memory for any n, so a query reads one sector and nothing else).
 * All layouts answer every query identically. */
#define QR_LAYOUT_BIRANK16    1
#define QR_LAYOUT_BIRANK64X2  2
#define QR_LAYOUT_QUADRANK16  3
#define QR_LAYOUT_QUADRANK64  4
#define QR_LAYOUT_BIRANK16X2  5
#define QR_LAYOUT_QUADRANK16X2 6
#define QR_LAYOUT_BIRANK32X2  7
typedef struct qr_fm qr_fm;         /* QuadFm: QuadRank over the BWT + C + spos + k-mer table */

/* ------------------------------------------------------------------ build */

/* BiRank16 (§3): 64-B lines j = [u16 b_j | 496 text bits], B = 496,
 * superblocks of S = 128 B bits with u32 s_i = floor(rank(iS) / 2^11) (line 407) and
 * b_j = rank(jB + 240) - 2^11 s_{j/128} (line 439).  Lines = floor(n/B)+1 (reading R4).
 * bits: packed text (host or device), ceil(n/64) words.  n < 2^43.  The build runs on
 * `device` (per-line popcount kernel, device-wide exclusive scan, inlining kernel). */
qr_status qr_birank_build(const uint64_t* bits, uint64_t n, int device, void* stream, qr_index** out);

/* QuadRank16 (§4; Listing 1): 64-B lines of four
 * u16 deltas b_{j,c} (u16 slots c + (c&2)) and B4 = 224 characters in transposed, negated
 * low/high bit planes; superblocks of 256 lines with u32 s_{i,c} = floor(rank(i S4, c)/2^13),
 * b_{j,c} = rank(j B4 + 96, c) - 2^13 s_{j/256, c}.  text2b: ceil(n/32) words.  n < 2^45. */
qr_status qr_quadrank_build(const uint64_t* text2b, uint64_t n, int device, void* stream, qr_index** out);

/* Build any layout: text is bits (BIRANK*) or 2-bit DNA (QUADRANK*), host or device, with the
 * conventions of qr_birank_build / qr_quadrank_build (which equal qr_build with layout
 * BIRANK16 / QUADRANK16).  n < 2^43 (BIRANK16), < 2^45 (QUADRANK16), < 2^48 (the 64-bit
 * variants).  QR_EINVAL for an unknown layout. */
qr_status qr_build(const uint64_t* text, uint64_t n, int layout, int device, void* stream, qr_index** out);

/* The layout of a handle (QR_LAYOUT_*). */
qr_status qr_layout(const qr_index* h, int* layout);

/* ------------------------------------------------------------------ queries */

/* out[k] = rank(q[k], c[k]) as u64, k < m.  Requires q[k] <= n; a larger q is a
 * contract violation: memory-safe (the line index is clamped), value unspecified.
 *   sigma = 4: c is required, c[k] in 0..3 (values are taken mod 4).
 *   sigma = 2: c may be NULL -> rank(q) (= rank(q,1)); else c[k] = 0 -> q - rank(q).
 * Per query: one 64-B line (one 32-B sector if q lies left of the block's anchor, else two)
 * plus one L2-resident superblock word (Eq. 1; Listing 1). */
qr_status qr_rank(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m, void* stream);

/* out4[4k + c] = rank(q[k], c) for c = 0..3 (rank_4).  sigma = 4
 * only (QR_EINVAL on a BiRank handle).  Output is 32 B per query, array-of-structs. */
qr_status qr_rank_all4(const qr_index* h, const uint64_t* q, uint64_t* out4, uint64_t m, void* stream);

/* Dependent-chain ("latency") mode (SPEC S:413 chaining rule; NEXT §8(f)4):
 * the m queries form chains of chain_len consecutive entries; inside a chain the i-th query
 * is q_eff = (q[i] + r_{i-1}) mod (n+1) with r_{-1} = 0, and out[i] = r_i = rank(q_eff, c[i])
 * (c as in qr_rank; NULL on sigma = 2 means rank(q)).  One thread walks each chain, so the time
 * per step is the latency of one dependent random gather.  Any layout; device pointers only. */
qr_status qr_rank_chain(const qr_index* h, const uint64_t* q, const uint8_t* c, uint64_t* out, uint64_t m,
                        uint64_t chain_len, void* stream);

/* ------------------------------------------------------------------ QuadFm */

/* Count-only FM index over a DNA text (App. D).  Builds the suffix
 * array of T$ on the GPU (prefix doubling over device radix sorts) unless sa_or_null gives
 * it (n+1 u32 entries, host or device), the BWT with '$' stored as A and its row spos kept
 * (lines 919-920), C[c] = 1 + #{t_i < c}, QuadRank16 over the n+1 BWT symbols, and the
 * k-mer interval table (line 918 uses 8-mers; the default width here depends on n, see
 * qr_fm_build_ex; key = 2 bits per char, last pattern char in the low bits).
 * text2b: ceil(n/32) words (host or device).  Requires 1 <= n and n + 1 < 2^32. */
qr_status qr_fm_build(const uint64_t* text2b, uint64_t n, const uint32_t* sa_or_null, int device, void* stream,
                      qr_fm** out);

/* As qr_fm_build from one byte per symbol (0..3 = A, C, G, T), the input form SURVEY §8(b)
 * proposes: text: n bytes (host or device), packed to 2 bits per symbol on the GPU.  A byte > 3
 * is QR_EINVAL (nothing is built).  Requires 1 <= n and n + 1 < 2^32. */
qr_status qr_fm_build_u8(const uint8_t* text, uint64_t n, const uint32_t* sa_or_null, int device, void* stream,
                         qr_fm** out);

/* As qr_fm_build with a k-mer seed table of width kmer_k (0..14; 0 = no table, every search
 * starts from [0, n+1)).  qr_fm_build picks the paper's 8 for n < 2^20, 10 for
 * n < 2^24 and, above, 11 when the BWT's rank layout plus the 32 MiB 11-mer table fit in 60% of
 * the device's L2 (seeds then come from L2), else 12 (on B200 the wider table
 * replaces more backward steps by one lookup); from n = 2^24 the approximate-search calls use a
 * 14-wide table of their own (2 GiB), built on the first such call (synchronous on its stream).  The table holds 4^kmer_k intervals (8 B each: 512 KiB at 8, 8 MiB at 10,
 * 128 MiB at 12, 2 GiB at 14).  Counts never depend on kmer_k.  QR_EINVAL outside 0..14. */
qr_status qr_fm_build_ex(const uint64_t* text2b, uint64_t n, const uint32_t* sa_or_null, int kmer_k, int device,
                         void* stream, qr_fm** out);

/* The k-mer table width of an FM handle. */
qr_status qr_fm_kmer_width(const qr_fm* fm, int* kmer_k);

/* As qr_fm_build_ex with the rank layout of the BWT: QR_LAYOUT_QUADRANK16 (the paper's QuadFm,
 * 2.29 bits/bp) or QR_LAYOUT_QUADRANK16X2 (the sector-local B200 variant, 33.4%: every rank of
 * a backward step reads one 32-B sector).  kmer_k = -1 takes qr_fm_build's
 * default width.  Counts never depend on either.  QR_EINVAL for another layout. */
qr_status qr_fm_build_opts(const uint64_t* text2b, uint64_t n, const uint32_t* sa_or_null, int kmer_k, int bwt_layout,
                           int device, void* stream, qr_fm** out);

/* out[k] = number of (overlapping) occurrences of pattern k in T, as u32 (backward search:
 * lo = C[c] + Occ(c, lo), hi = C[c] + Occ(c, hi), Occ(c,x) = rank(x,c) - [c = A and x > spos];
 * seeded by the k-mer table when the pattern has >= K symbols).  patterns: concatenated, one
 * byte per symbol (0..3, taken mod 4).  lengths: u32[m], pattern k starts at the exclusive
 * prefix sum of lengths (computed on the device); or lengths = NULL and every pattern has
 * fixed_len symbols.  An empty pattern counts n + 1.  Patterns are counted as given (no
 * reverse complement: that is a second call).  The kernel reads pattern bytes in
 * aligned 8-byte words, so it may read up to 7 bytes past the last pattern inside the same
 * 8-byte-aligned word (never across an allocation: such a word always holds a valid byte). */
qr_status qr_fm_count(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths, uint32_t fixed_len,
                      uint32_t* out, uint64_t m, void* stream);

/* Both strands in one launch (reads are counted "in both forward and
 * reverse-complement direction"; NEXT §8(f)1): out_fwd[k] = count of pattern k,
 * out_rc[k] = count of its reverse complement RC(P)[j] = 3 - P[len-1-j] (A<->T, C<->G,
 * reversed).  The reverse complement is read from the same bytes inside the kernel (no copy).
 * Arguments and memory spaces as qr_fm_count. */
qr_status qr_fm_count_both(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths, uint32_t fixed_len,
                           uint32_t* out_fwd, uint32_t* out_rc, uint64_t m, void* stream);

/* Approximate counting (NEXT §8(f)3; rank_4's motivation): out[k] = number of
 * text positions where pattern k matches with at most max_mismatches substitutions (Hamming
 * distance; 0..3 — QR_EINVAL otherwise; 0 is qr_fm_count).  max_mismatches = 1 branches on
 * every pattern position with one rank_4 at lo and one at hi (the four extensions of the exact
 * interval) and reads the 3K single-substitution variants of the last K symbols from the k-mer
 * table.  2 and 3 backtrack from the full interval with rank_4 at every node (one frame per
 * mismatch level, no seeding); their work grows steeply with the pattern length and k.
 * Arguments and memory spaces as qr_fm_count. */
qr_status qr_fm_count_approx(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths, uint32_t fixed_len,
                             uint32_t max_mismatches, uint32_t* out, uint64_t m, void* stream);

/* Both strands of every pattern within max_mismatches substitutions (0..3), in one launch:
 * out_fwd[k] as qr_fm_count_approx, out_rc[k] the same count for the reverse complement
 * RC(P)[j] = 3 - P[len-1-j] (read from the same bytes, never materialised) —
 * the paper's read workload with its 1% substitutions.  Arguments as
 * qr_fm_count_approx; out_rc: u32[m], same memory space as out_fwd. */
qr_status qr_fm_count_approx_both(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths,
                                  uint32_t fixed_len, uint32_t max_mismatches, uint32_t* out_fwd, uint32_t* out_rc,
                                  uint64_t m, void* stream);

/* As qr_fm_count (device pointers only), additionally accumulating into work[0] the number of
 * backward steps executed after seeding and into work[1] the number of distinct 64-B lines
 * those steps touch (1 or 2 per step) — the algorithmic-bytes denominator of SURVEY §8(d).
 * work: 2 u64 on the device, accumulated (not reset). */
qr_status qr_fm_count_work(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths, uint32_t fixed_len,
                           uint32_t* out, uint64_t m, uint64_t* work, void* stream);

/* Work accounting of every count flavour (device pointers only): the call qr_fm_count_approx
 * (max_mismatches 0..3; 0 = exact) or, with out_rc non-NULL, qr_fm_count_approx_both makes,
 * accumulating into work[0] the rank evaluations at an interval's two ends (exact backward
 * steps after seeding, rank_4 pairs of the search tree) plus k-mer table
 * lookups, and into work[1] the distinct 64-B lines (table entries) they gather — the
 * denominator of the FM roofline fraction.  For max_mismatches = 0 and one
 * strand this is qr_fm_count_work.  work: 2 u64 on the device, accumulated (not reset). */
qr_status qr_fm_count_work_ex(const qr_fm* fm, const uint8_t* patterns, const uint32_t* lengths, uint32_t fixed_len,
                              uint32_t max_mismatches, uint32_t* out_fwd, uint32_t* out_rc, uint64_t m,
                              uint64_t* work, void* stream);

/* ------------------------------------------------------------------ measurement */

/* Gather ceiling ("null rank"): the same q stream, the same line-index
 * arithmetic and the same loads as qr_rank, no popcount and no superblock read;
 * out[k] = XOR of the loaded words.  mode 0: exactly the sectors qr_rank reads (32 B or
 * 64 B); mode 1: the full 64-B line always; mode 2: mode 0 plus qr_rank's superblock-word
 * read (BiRank; on QuadRank mode 2 = mode 0); mode 3: the cluster shared-memory rank kernel's
 * own launch shape and loads without the superblock read (BiRank16 with a superblock cache,
 * qr_super_cache_bytes > 0; else QR_EINVAL); mode 4: mode 0's loads with rank_4's output shape,
 * 32 B written per query (QuadRank16 only; out holds 4m u64).  Device pointers only. */
qr_status qr_gather_ceiling(const qr_index* h, const uint64_t* q, uint64_t* out, uint64_t m, int mode, void* stream);

/* ------------------------------------------------------------------ handles */

/* sigma (2 or 4), n, and the layout's device bytes (lines + superblock array). */
qr_status qr_info(const qr_index* h, uint64_t* n, int* sigma, uint64_t* line_bytes, uint64_t* super_bytes);

/* Bytes of the re-encoded superblock table that the cluster rank kernels keep in shared
 * memory (2 CTAs x *cta_bytes; sbcache.cu), or 0 when this handle has no 2-CTA
 * table (layouts without an L1 array, n >= 2^35, or a table larger than two CTAs' shared
 * memory: large BiRank16 / QuadRank16 handles then use a 4/8/16-CTA cluster table for batches
 * >= 2^22, else global memory).  A cache of s_i / s_{i,c}:
 * results never depend on it. */
qr_status qr_super_cache_bytes(const qr_index* h, uint64_t* cta_bytes);
/* Number of 2-CTA clusters those kernels launch (as many as fit at once; 0 without a cache). */
qr_status qr_super_cache_clusters(const qr_index* h, int* clusters);

/* Copy the layout to buffers of qr_info's sizes (host, or device — e.g. to broadcast a built
 * structure to other GPUs; either may be NULL).  Synchronous. */
qr_status qr_export_layout(const qr_index* h, void* host_lines, void* host_super);

/* Re-create a handle from a layout saved with qr_export_layout (checkpoint / resume without
 * rebuilding; builds are deterministic): lines and super are host or device buffers of
 * line_bytes and super_bytes bytes, which must equal the sizes qr_info reports for (n, layout)
 * (else QR_EINVAL: a truncated file or a mismatched n is rejected before any copy); super may be
 * NULL (super_bytes 0) for layouts without an L1 array.  The contents are trusted (no
 * validation pass over the words). */
qr_status qr_import_layout(const void* lines, uint64_t line_bytes, const void* super, uint64_t super_bytes, uint64_t n,
                           int layout, int device, void* stream, qr_index** out);

/* n, N = n+1 BWT rows, spos, C[0..4] (C[4] = n+1), and the QuadRank handle over the BWT
 * (owned by fm; valid until qr_fm_free). */
qr_status qr_fm_info(const qr_fm* fm, uint64_t* n, uint64_t* spos, uint64_t C[5], const qr_index** bwt_rank);

/* Copy the k-mer interval table (4^kmer_k pairs of u32 [lo, hi); 65536 for the default
 * width 8) to a host buffer. Synchronous. */
qr_status qr_fm_export_kmer(const qr_fm* fm, uint32_t* host_pairs);

/* Replicate a handle onto another device (peer copy over NVLink when available). */
qr_status qr_clone_to_device(const qr_index* h, int device, void* stream, qr_index** out);
qr_status qr_fm_clone_to_device(const qr_fm* fm, int device, void* stream, qr_fm** out);

/* Synchronise `stream` and surface any asynchronous error. */
qr_status qr_sync(void* stream);

/* Output checksum for multi-GPU verification ("all_reduce of a u64 checksum"):
 * *sum (one u64 on the device, accumulated, not reset) += sum over i < count of
 * mix(index0 + i, word_i) mod 2^64, where word_i is element i of `data` (word_bytes 4 or 8) and
 * mix a 64-bit hash of (global index, value).  The sum is additive over disjoint index ranges,
 * so shards checksummed on different GPUs add up (one all_reduce) to the checksum of the whole
 * batch on one GPU.  Not part of the method; measurement utility.  Device pointers only; QR_EINVAL
 * for another word size. */
qr_status qr_checksum(const void* data, uint64_t count, int word_bytes, uint64_t index0, uint64_t* sum, void* stream);

void qr_free(qr_index* h);
void qr_fm_free(qr_fm* fm);

/* Thread-local message of the last failure on this thread ("" if none). */
const char* qr_last_error(void);

/* Process-wide launch-configuration knobs for measurement sweeps.  Results never depend on
 * them; they are not synchronised (set them before issuing work from other threads).
 * QR_EINVAL for an unknown key or an out-of-range value.
 *
 * Rank kernel shape:
 *   "rank_pair"        0 one lane per query, 1 lane pairs, 2 (default) by structure size: one
 *                      lane per query while the line array fits 0.6 x L2, lane pairs up to
 *                      2.2 x L2, the cluster kernel beyond.
 *   "rank_lane_table"  1 (default): the one-lane kernels read the superblock words from a
 *                      per-CTA shared-memory copy of the packed table when it is <= 32 KB; 0: L2.
 *   "rank_resident"    1 (default): BiRank16 / QuadRank16 structures whose lines and table fit
 *                      one CTA's shared memory (<= 200 KB, e.g. configs[0]) are copied into every
 *                      CTA of a one-CTA-per-SM grid and queried from there (lines swizzled over
 *                      the banks), for batches whose 16 B/query of I/O is >= 2x the bytes all
 *                      the copies read; 0: lines from L2.
 *   "rank_big_pack"    1: also build the large-n superblock table for handles built afterwards
 *                      (normally only when the 2-CTA table cannot be used: BiRank16 2^35 <= n <
 *                      2^37, the 6-superblock groups with 24-bit bases + three high-bit group
 *                      boundaries, <= 184 KB per CTA; QuadRank16 ~2^32.6 < n < 2^35 chars, the
 *                      8-superblock groups, <= 184 KB per CTA; split over a 4/8/16-CTA
 *                      cluster) — for tests.
 *   "rank_big_cs"      0 (default): the smallest cluster size meeting that bound; 4, 8, 16: force.
 *   "rank_smem"        the 2-CTA cluster shared-memory kernels: 0 never, 1 (default) by
 *                      structure size for batches >= 2^22, 2 whenever the table exists.
 *   "rank_s_lane"      global lane-pair kernels: which lane of a pair loads the superblock word.
 *   "index64"          1: always the 64-bit line-index path that n >= 2^36 (sigma=2) / 2^37
 *                      (sigma=4) selects, so that it can be tested on small n.
 * Rank launch configuration:
 *   "rank_k"           1, 2, 4, 8: queries per thread (lane pair) per iteration, global kernels.
 *   "rank_blocks_per_sm", "fm_blocks_per_sm"  1..64: 256-thread CTAs per SM of the static
 *                      (multi-wave, grid-stride) order.
 *   "rank_dyn"         1 (default): batches >= 2^22 take work in chunks from a global counter
 *                      on a resident grid; 0: the static grid-stride order.
 *   "rank_smem_k"      cluster kernels' queries per lane pair: 0 auto (BiRank 4, QuadRank 2),
 *                      1-4 with 1024-thread CTAs, 6 with 768, 8 with 512 (resets the next knob).
 *   "rank_smem_threads"  cluster kernels' CTA size for the current K (1024 for K 1-4, 768 for
 *                      K 4 or 6, 512 for K 8; 0 = the default for K).
 *   "rank_smem_clusters" 0: as many 2-CTA clusters as fit at once, else that many.
 *   "l2_fetch_granularity"  cudaLimitMaxL2FetchGranularity of the current device (bytes).
 * QuadFm:
 *   "fm_step"          0 auto by L2 residency of the BWT layout, 1 line-de-duplicating step,
 *                      2 lean step.
 *   "fm_dyn"           1 (default): persistent grid, warps take pattern chunks from a global
 *                      counter; 0: static grid stride.
 *   "fm_seed"          k-mer seeds by a parallel pre-pass: 0 auto (BWT layout fits half the
 *                      L2), 1 never, 2 always.
 *   "fm_smem"          superblock words of the count kernel from shared memory: 0 off, 1 auto
 *                      (the raw array or the packed table when either fits 48 KB per CTA), 2 the
 *                      packed table whenever it fits a CTA.
 * Staged host-pointer path:
 *   "stage_chunk"      queries per chunk (>= 1024);  "stage_slots"  2..4 buffers / streams. */
qr_status qr_set_tuning(const char* key, int64_t value);

/* Library version string. */
const char* qr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QRANK_H */
