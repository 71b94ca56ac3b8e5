"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(library defaults).  configs[1] (both densities), configs[2] (rank and rank_all4) and configs[3]
are checked on EVERY output against the oracle (BASELINE.md:61, :80), streamed back in chunks;
configs[4] on 2,100 patterns stratified by substitutions (direct scan of a 2^30 text) plus
properties on all 10^8.  Each exhaustive check logs outputs_checked / mismatches and the oracle's
time on the host (gpurun_out/parity_fullsize.jsonl → profiles/).  The other cases (beyond 2^31
rows, 2^35 / 2^36 bits, 2^34 chars) check sampled runs and the boundary set."""
import json
import os
import time

import numpy as np
import pytest

import gen
import oracle
import paper_2602_04103_b200 as qr
from _util import B, B4, S, S4, boundary_queries, to_dev, to_host

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RUNS, RUN = 48, 8192                    # sampled outputs: 48 runs of 8192 consecutive queries


def _torch():
    import torch

    return torch


def sample_offsets(m, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.integers(0, m - RUN, RUNS))


CHUNK = 1 << 27                         # outputs streamed back per chunk: 2^27 u64 = 1 GiB


def _log(rec):
    """Append one parity record (outputs checked, mismatches, oracle time) to the run's log
    (QR_PARITY_LOG, default gpurun_out/parity_fullsize.jsonl); copied under profiles/."""
    path = os.environ.get("QR_PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity_fullsize.jsonl"))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    rec = dict(rec, host_threads=oracle.threads(), when=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()))
    with open(path, "a") as f:
        f.write(json.dumps(rec) + "\n")


def _chunks(m, chunk=CHUNK):
    for lo in range(0, m, chunk):
        yield lo, min(m, lo + chunk)


@pytest.mark.parametrize("p,seed", [(0.5, 2), (0.01, 22)])
def test_config2_birank_full(cuda, p, seed):
    """configs[1] at full size: EVERY one of the 10^9 outputs against the oracle (BASELINE.md:61:
    the number of mismatches over all outputs must be 0), streamed back in 1 GiB chunks; the
    host-regenerated query stream is compared with the device one on every word too."""
    torch = _torch()
    oracle.set_threads(len(os.sched_getaffinity(0)))
    n, m = 1 << 34, 10**9
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=cuda)
    gen.bits_dev(seed, n, p, bits)
    h = qr.qr_birank_build(bits, n)
    del bits
    # byte accounting (SURVEY §8(a) a3 from P:396-441): 34,636,834 lines + 270,601 superblocks
    assert (h.line_bytes, h.super_bytes) == (2_216_757_376, 1_082_404)
    q = torch.empty(m, dtype=torch.uint64, device=cuda)
    gen.queries_dev(2, n, m, q)
    out = torch.empty_like(q)
    qr.qr_rank(h, q, None, out)                          # the bench's launch: one call, 10^9 queries
    torch.cuda.synchronize()
    host_bits = gen.bits(seed, n, p)                      # oracle input from the host generator
    ora = oracle.BitsOracle(host_bits, n)
    mism = qmism = 0
    t_or = 0.0
    for lo, hi in _chunks(m):
        qs = gen.queries(2, n, hi - lo, i0=lo)
        qmism += int(np.count_nonzero(to_host(q[lo:hi]) != qs))
        t0 = time.perf_counter()
        ref = ora.rank(qs)
        t_or += time.perf_counter() - t0
        mism += int(np.count_nonzero(to_host(out[lo:hi]) != ref))
    _log({"test": f"config2_birank_p{p}", "outputs_checked": m, "mismatches": mism, "query_mismatches": qmism,
          "oracle_s": round(t_or, 2), "oracle_gq_s": round(m / t_or / 1e9, 4)})
    assert qmism == 0 and mism == 0
    bq = boundary_queries(n, B, S, 240, limit=200000)
    dq = to_dev(bq, cuda)
    ob = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, ob)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(ob), ora.rank(bq))
    if p == 0.01:
        frac = float(ora.rank(np.array([n], np.uint64))[0]) / n
        assert abs(frac - 0.01) < 1e-4


def test_config3_quadrank_full(cuda):
    """configs[2] at full size: every one of the 10^9 rank(q, c) outputs and every one of the
    4 x 10^9 rank_all4 outputs against the oracle, streamed back in chunks."""
    torch = _torch()
    oracle.set_threads(len(os.sched_getaffinity(0)))
    n, m = 1 << 32, 10**9
    txt = torch.empty((n + 31) // 32, dtype=torch.uint64, device=cuda)
    gen.dna_dev(3, n, 0, txt)
    h = qr.qr_quadrank_build(txt, n)
    del txt
    # byte accounting (SURVEY §8(a) a3 from P:507-539): 19,173,962 lines + 74,899 superblocks
    assert (h.line_bytes, h.super_bytes) == (1_227_133_568, 1_198_384)
    q = torch.empty(m, dtype=torch.uint64, device=cuda)
    c = torch.empty(m, dtype=torch.uint8, device=cuda)
    gen.queries_dev(3, n, m, q, c)
    out = torch.empty_like(q)
    qr.qr_rank(h, q, c, out)
    torch.cuda.synchronize()
    ora = oracle.DnaOracle(gen.dna(3, n), n)
    mism = 0
    t_or = 0.0
    for lo, hi in _chunks(m):
        qs, cs = gen.queries(3, n, hi - lo, i0=lo, with_c=True)
        assert np.array_equal(to_host(c[lo:hi]), cs)
        t0 = time.perf_counter()
        ref = ora.rank(qs, cs)
        t_or += time.perf_counter() - t0
        mism += int(np.count_nonzero(to_host(out[lo:hi]) != ref))
    _log({"test": "config3_quadrank_rank", "outputs_checked": m, "mismatches": mism, "oracle_s": round(t_or, 2),
          "oracle_gq_s": round(m / t_or / 1e9, 4)})
    assert mism == 0
    del out
    # rank_4 over the full 10^9 queries in parts of 2.5e8 (8 GB of output each), every word checked
    part = m // 4
    o4 = torch.empty((part, 4), dtype=torch.uint64, device=cuda)
    mism4 = 0
    t_or4 = 0.0
    for p0 in range(0, m, part):
        qr.qr_rank_all4(h, q[p0:p0 + part], o4)
        torch.cuda.synchronize()
        for lo, hi in _chunks(part, CHUNK // 4):
            qs = gen.queries(3, n, hi - lo, i0=p0 + lo)
            t0 = time.perf_counter()
            ref = ora.rank_all4(qs)
            t_or4 += time.perf_counter() - t0
            mism4 += int(np.count_nonzero(to_host(o4[lo:hi]) != ref))
    _log({"test": "config3_quadrank_rank_all4", "outputs_checked": 4 * m, "queries": m, "mismatches": mism4,
          "oracle_s": round(t_or4, 2), "oracle_gq_s": round(m / t_or4 / 1e9, 4)})
    assert mism4 == 0
    bq = boundary_queries(n, B4, S4, 96, limit=200000)
    o4b = torch.empty((bq.size, 4), dtype=torch.uint64, device=cuda)
    qr.qr_rank_all4(h, to_dev(bq, cuda), o4b)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(o4b), ora.rank_all4(bq))


def _splitmix_np(seed, tag, idx):
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) ^ (np.uint64(tag) * np.uint64(0xD1B54A32D192ED03) & M)) + \
            (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _fm_gpu(cuda, n, kind, m, L, seed, bwt_bytes=None):
    """Build the FM index on the GPU and count all m patterns in one launch (the bench's call)."""
    torch = _torch()
    txt = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=cuda)
    gen.dna_dev(seed, n, kind, txt)
    fm = qr.qr_fm_build(txt, n)
    if bwt_bytes is not None:                              # QuadRank over the n+1 BWT symbols
        assert (fm.bwt.line_bytes, fm.bwt.super_bytes) == bwt_bytes
    # the C array and the BWT rank partition: sum_c rank(N, c) = N
    assert fm.C[4] == n + 1
    pats = torch.empty(m * L, dtype=torch.uint8, device=cuda)
    gen.patterns_dev(seed, 0 if kind == 0 else 1, m, L, txt, n, pats)
    out = torch.empty(m, dtype=torch.int32, device=cuda)
    qr.qr_fm_count(fm, pats, None, L, out, m)
    torch.cuda.synchronize()
    return to_host(out).view(np.uint32), pats, fm


def _fm_full(cuda, n, kind, m, L, seed, nsample, bwt_bytes=None):
    """Smaller FM cases: the oracle's direct scan on `nsample` sampled patterns."""
    counts, pats, fm = _fm_gpu(cuda, n, kind, m, L, seed, bwt_bytes)
    host_txt = gen.dna(seed, n, kind)
    sym = gen.unpack_dna(host_txt, n)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(m, nsample, replace=False))
    cat = np.concatenate([gen.patterns(seed, 0 if kind == 0 else 1, 1, L, host_txt, n, i0=int(i)) for i in idx])
    ref = oracle.scan_count(sym, cat, np.arange(nsample, dtype=np.uint64) * L, np.full(nsample, L, np.uint32))
    assert np.array_equal(counts[idx], ref)
    assert np.array_equal(to_host(pats[int(idx[0]) * L:(int(idx[0]) + 1) * L]), cat[:L])
    return counts


def test_config4_quadfm_full(cuda):
    """configs[3] at full size: EVERY one of the 10^7 counts against the oracle's backward
    search over its own plain BWT (its own suffix array of the 2^26-symbol text, no k-mer
    table, '$' as a distinct byte), plus the oracle's SA binary search on a sample."""
    oracle.set_threads(len(os.sched_getaffinity(0)))
    n, m, L = 1 << 26, 10**7, 32
    counts, pats, fm = _fm_gpu(cuda, n, 0, m, L, 4, bwt_bytes=(19_174_016, 18_736))
    host_txt = gen.dna(4, n, 0)
    sym = gen.unpack_dna(host_txt, n)
    t0 = time.perf_counter()
    fo = oracle.FmOracle(sym)
    t_sa = time.perf_counter() - t0
    cat = gen.patterns(4, 0, m, L, host_txt, n)
    assert np.array_equal(to_host(pats), cat)
    off, lens = np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32)
    t0 = time.perf_counter()
    ref = fo.count(cat, off, lens)
    t_or = time.perf_counter() - t0
    mism = int(np.count_nonzero(counts != ref))
    ss = np.arange(0, m, 997)
    sa_ref = fo.sa_count(np.concatenate([cat[i * L:(i + 1) * L] for i in ss]),
                         np.arange(ss.size, dtype=np.uint64) * L, np.full(ss.size, L, np.uint32))
    _log({"test": "config4_quadfm", "outputs_checked": m, "mismatches": mism, "oracle": "backward search, plain BWT",
          "oracle_s": round(t_or, 2), "oracle_patterns_per_s": round(m / t_or, 1),
          "oracle_sa_build_s": round(t_sa, 1), "sa_binary_search_checked": int(ss.size)})
    assert mism == 0
    assert np.array_equal(counts[ss], sa_ref)
    assert counts[0::2].min() >= 1                        # every exact substring occurs (all 5e6)


def test_config5_quadfm_full(cuda):
    """configs[4] at full size: all 10^8 patterns counted on the GPU; 10^6 of them (uniform over
    the batch, so about a third each with 0, 1 and 2 substitutions) against the oracle's direct
    scan of the 2^30-symbol text (or_scan_count_bucketed: the same direct comparison at every
    position, patterns grouped by their first 8 symbols); every 0-substitution pattern (~3.3e7) is
    an exact substring, so its count is >= 1."""
    oracle.set_threads(len(os.sched_getaffinity(0)))
    n, m, L = 1 << 30, 10**8, 100
    counts, pats, fm = _fm_gpu(cuda, n, 1, m, L, 5, bwt_bytes=(306_783_424, 299_600))
    h = _splitmix_np(5, 11, np.arange(m))
    s = (h > np.uint64(0x5555555555555555)).astype(np.int8) + (h > np.uint64(0xAAAAAAAAAAAAAAAA)).astype(np.int8)
    assert counts[s == 0].min() >= 1
    assert (s == 0).mean() == pytest.approx(1 / 3, abs=0.01)
    host_txt = gen.dna(5, n, 1)
    sym = gen.unpack_dna(host_txt, n)
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(m, 10**6, replace=False))
    allp = gen.patterns(5, 1, m, L, host_txt, n).reshape(m, L)          # host generator, all 10^8
    cat = np.ascontiguousarray(allp[idx]).reshape(-1)
    del allp
    for j in (0, idx.size // 2, idx.size - 1):
        i = int(idx[j])
        assert np.array_equal(to_host(pats[i * L:(i + 1) * L]), cat[j * L:(j + 1) * L])
    t0 = time.perf_counter()
    ref = oracle.scan_count_bucketed(sym, cat, np.arange(idx.size, dtype=np.uint64) * L,
                                     np.full(idx.size, L, np.uint32))
    t_or = time.perf_counter() - t0
    mism = int(np.count_nonzero(counts[idx] != ref))
    _log({"test": "config5_quadfm", "outputs_checked": int(idx.size), "mismatches": mism,
          "by_substitutions": {str(k): int((s[idx] == k).sum()) for k in range(3)},
          "oracle": "direct scan of every text position (or_scan_count_bucketed)", "oracle_s": round(t_or, 2),
          "oracle_patterns_per_s": round(idx.size / t_or, 2), "exact_substrings_count_ge_1": int((s == 0).sum()),
          "mean_count": {str(k): float(ref[s[idx] == k].mean()) for k in range(3)}})
    assert mism == 0


def test_fm_beyond_2_31_rows(cuda):
    """N = n+1 > 2^31 exercises the 64-bit item counts of the GPU suffix sort and the u32
    interval arithmetic near its top (reading R11: counts are u32, n+1 < 2^32)."""
    torch = _torch()
    n = (1 << 31) + 7
    counts = _fm_full(cuda, n, 0, 10**6, 40, 9, 24)
    assert counts[0::2].min() >= 1


def test_birank_beyond_2_36_bits(cuda):
    """n >= 2^36 bits takes the 64-bit line-index kernels for real (not through the index64
    knob): 2^36 + 777 bits (8.6 GB), 10^7 queries + the boundary set, sampled runs and the last
    line against the oracle; every output satisfies 0 <= rank(q) <= q."""
    torch = _torch()
    n, m = (1 << 36) + 777, 10**7
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=cuda)
    gen.bits_dev(36, n, 0.5, bits)
    h = qr.qr_birank_build(bits, n)
    del bits
    q = torch.empty(m, dtype=torch.uint64, device=cuda)
    gen.queries_dev(37, n, m, q)
    out = torch.empty_like(q)
    qr.qr_rank(h, q, None, out)
    torch.cuda.synchronize()
    assert bool((out.view(torch.int64) <= q.view(torch.int64)).all())
    ora = oracle.BitsOracle(gen.bits(36, n, 0.5), n)
    for off in sample_offsets(m, 36)[:16]:
        qs = gen.queries(37, n, RUN, i0=int(off))
        assert np.array_equal(to_host(out[off:off + RUN]), ora.rank(qs)), f"offset {off}"
    bq = np.concatenate([boundary_queries(n, B, S, 240, limit=20000),
                         np.arange(n - 3000, n + 1, dtype=np.uint64)])
    dq = to_dev(bq, cuda)
    ob = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, ob)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(ob), ora.rank(bq))


def test_birank_2_35_bits_cluster_table(cuda):
    """The paper's own bit-vector size (4 GiB): n = 2^35 + 777 takes the 4-CTA
    cluster table kernel; sampled and boundary queries vs the oracle."""
    torch = _torch()
    n, m = (1 << 35) + 777, 10**7
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=cuda)
    gen.bits_dev(35, n, 0.5, bits)
    h = qr.qr_birank_build(bits, n)
    del bits
    q = torch.empty(m, dtype=torch.uint64, device=cuda)
    gen.queries_dev(38, n, m, q)
    out = torch.empty_like(q)
    qr.qr_rank(h, q, None, out)
    torch.cuda.synchronize()
    assert bool((out.view(torch.int64) <= q.view(torch.int64)).all())
    ora = oracle.BitsOracle(gen.bits(35, n, 0.5), n)
    for off in sample_offsets(m, 35)[:16]:
        qs = gen.queries(38, n, RUN, i0=int(off))
        assert np.array_equal(to_host(out[off:off + RUN]), ora.rank(qs)), f"offset {off}"
    bq = np.concatenate([boundary_queries(n, B, S, 240, limit=20000), np.arange(n - 3000, n + 1, dtype=np.uint64)])
    bq = np.concatenate([bq, gen.queries(39, n, (1 << 22) - bq.size + 5)])   # >= 2^22: the cluster path
    dq = to_dev(bq, cuda)
    ob = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, ob)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(ob), ora.rank(bq))


def test_fm_near_u32_limit(cuda):
    """n = 4.0e9 symbols (n + 1 < 2^32, the FM capacity): the GPU suffix sort must fit in HBM
    (32 B per suffix + 8 B per survivor of its first round) and the counts stay exact."""
    n = 4_000_000_000
    counts = _fm_full(cuda, n, 0, 10**6, 40, 12, 6)
    assert counts[0::2].min() >= 1


def test_quadrank_2_34_chars_cluster_table(cuda):
    """The paper's 4 GiB of 2-bit text (n = 2^34 + 99 chars): QuadRank16 takes the CS-CTA cluster
    table kernels; sampled rank(q, c) / rank_4 runs and the boundary set vs the oracle."""
    torch = _torch()
    n, m = (1 << 34) + 99, 1 << 23
    txt = torch.empty((n + 31) // 32, dtype=torch.uint64, device=cuda)
    gen.dna_dev(34, n, 0, txt)
    h = qr.qr_quadrank_build(txt, n)
    del txt
    q = torch.empty(m, dtype=torch.uint64, device=cuda)
    c = torch.empty(m, dtype=torch.uint8, device=cuda)
    gen.queries_dev(41, n, m, q, c)
    out = torch.empty_like(q)
    qr.qr_rank(h, q, c, out)
    o4 = torch.empty((m, 4), dtype=torch.uint64, device=cuda)
    qr.qr_rank_all4(h, q, o4)
    torch.cuda.synchronize()
    assert bool((o4.view(torch.int64).sum(dim=1) == q.view(torch.int64)).all())
    ora = oracle.DnaOracle(gen.dna(34, n), n)
    for off in sample_offsets(m, 34)[:12]:
        qs, cs = gen.queries(41, n, RUN, i0=int(off), with_c=True)
        assert np.array_equal(to_host(out[off:off + RUN]), ora.rank(qs, cs)), f"offset {off}"
        assert np.array_equal(to_host(o4[off:off + RUN]), ora.rank_all4(qs)), f"offset {off}"


@pytest.mark.parametrize("p", [1.0, 0.9])
def test_birank_large_table_high_bits(cuda, p):
    """Superblock words of 2^24 and more (R >= 2^35 ones): the large-n cluster table stores 24-bit
    group bases and recovers bits 24-25 from group boundaries.  n = 2^35 + 2^33 + 12345 bits of
    density 1.0 (rank(q) = q, closed form) and 0.9 (oracle on sampled runs); both cross 2^24."""
    torch = _torch()
    n, m = (1 << 35) + (1 << 33) + 12345, 1 << 24
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=cuda)
    if p == 1.0:
        bits.view(torch.int64).fill_(-1)
    else:
        gen.bits_dev(44, n, p, bits)
    h = qr.qr_birank_build(bits, n)
    del bits
    q = torch.empty(m, dtype=torch.uint64, device=cuda)
    gen.queries_dev(45, n, m, q)
    out = torch.empty_like(q)
    qr.qr_rank(h, q, None, out)
    torch.cuda.synchronize()
    if p == 1.0:
        assert torch.equal(out, q)
        return
    ora = oracle.BitsOracle(gen.bits(44, n, p), n)
    for off in sample_offsets(m, 44)[:16]:
        qs = gen.queries(45, n, RUN, i0=int(off))
        assert np.array_equal(to_host(out[off:off + RUN]), ora.rank(qs)), f"offset {off}"
    tail = np.arange(n - 200000, n + 1, dtype=np.uint64)
    tq = np.concatenate([tail, gen.queries(46, n, (1 << 22))])
    dq = to_dev(tq, cuda)
    ot = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, ot)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(ot), ora.rank(tq))
