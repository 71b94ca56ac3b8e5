"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(library defaults).  The GPU computes every output of the full batch; the oracle checks
sampled outputs one by one (contiguous runs at seeded offsets + the boundary set), and
properties that hold at any size are checked on all outputs."""
import numpy as np
import pytest

import gen
import oracle
import paper_2602_04103_b200 as qr
from _util import B, B4, S, S4, boundary_queries, to_dev, to_host

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RUNS, RUN = 48, 8192                    # sampled outputs: 48 runs of 8192 consecutive queries


def _torch():
    import torch

    return torch


def sample_offsets(m, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.integers(0, m - RUN, RUNS))


@pytest.mark.parametrize("p,seed", [(0.5, 2), (0.01, 22)])
def test_config2_birank_full(cuda, p, seed):
    torch = _torch()
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
    qr.qr_rank(h, q, None, out)
    torch.cuda.synchronize()
    # any-size property on all outputs: 0 <= rank(q) <= q
    assert bool((out.view(torch.int64) <= q.view(torch.int64)).all())
    host_bits = gen.bits(seed, n, p)                      # oracle input from the host generator
    ora = oracle.BitsOracle(host_bits, n)
    for off in sample_offsets(m, seed):
        qs = gen.queries(2, n, RUN, i0=int(off))
        assert np.array_equal(to_host(q[off:off + RUN]), qs)   # device and host streams agree
        assert np.array_equal(to_host(out[off:off + RUN]), ora.rank(qs)), f"offset {off}"
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
    torch = _torch()
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
    assert bool((out.view(torch.int64) <= q.view(torch.int64)).all())
    ora = oracle.DnaOracle(gen.dna(3, n), n)
    for off in sample_offsets(m, 3):
        qs, cs = gen.queries(3, n, RUN, i0=int(off), with_c=True)
        assert np.array_equal(to_host(out[off:off + RUN]), ora.rank(qs, cs)), f"offset {off}"
    # rank_4 over the full 10^9 queries (chunks of 2.5e8 to bound memory); sum_c = q on all
    o4 = torch.empty((m // 4, 4), dtype=torch.uint64, device=cuda)
    for part in range(4):
        lo = part * (m // 4)
        qr.qr_rank_all4(h, q[lo:lo + m // 4], o4)
        torch.cuda.synchronize()
        assert bool((o4.view(torch.int64).sum(dim=1) == q[lo:lo + m // 4].view(torch.int64)).all())
        if part == 1:
            for off in sample_offsets(m // 4, 33)[:12]:
                qs = gen.queries(3, n, RUN, i0=int(lo + off))
                assert np.array_equal(to_host(o4[off:off + RUN]), ora.rank_all4(qs))
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


def _fm_full(cuda, n, kind, m, L, seed, nsample, bwt_bytes=None):
    torch = _torch()
    txt = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=cuda)
    gen.dna_dev(seed, n, kind, txt)
    fm = qr.qr_fm_build(txt, n)
    if bwt_bytes is not None:                              # QuadRank over the n+1 BWT symbols
        assert (fm.bwt.line_bytes, fm.bwt.super_bytes) == bwt_bytes
    pats = torch.empty(m * L, dtype=torch.uint8, device=cuda)
    gen.patterns_dev(seed, 0 if kind == 0 else 1, m, L, txt, n, pats)
    out = torch.empty(m, dtype=torch.int32, device=cuda)
    qr.qr_fm_count(fm, pats, None, L, out, m)
    torch.cuda.synchronize()
    counts = to_host(out).view(np.uint32)
    host_txt = gen.dna(seed, n, kind)
    sym = gen.unpack_dna(host_txt, n)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(m, nsample, replace=False))
    cat = np.concatenate([gen.patterns(seed, 0 if kind == 0 else 1, 1, L, host_txt, n, i0=int(i)) for i in idx])
    ref = oracle.scan_count(sym, cat, np.arange(nsample, dtype=np.uint64) * L, np.full(nsample, L, np.uint32))
    assert np.array_equal(counts[idx], ref)
    assert np.array_equal(to_host(pats[int(idx[0]) * L:(int(idx[0]) + 1) * L]), cat[:L])
    # the C array and the BWT rank partition: sum_c rank(N, c) = N
    assert fm.C[4] == n + 1
    return counts


def test_config4_quadfm_full(cuda):
    n, m, L = 1 << 26, 10**7, 32
    counts = _fm_full(cuda, n, 0, m, L, 4, 256, bwt_bytes=(19_174_016, 18_736))
    assert counts[0::2].min() >= 1                        # every exact substring occurs (all 5e6)


def test_config5_quadfm_full(cuda):
    n, m, L = 1 << 30, 10**8, 100
    counts = _fm_full(cuda, n, 1, m, L, 5, 48, bwt_bytes=(306_783_424, 299_600))
    # patterns drawn with 0 substitutions are exact substrings: count >= 1 (all of them)
    s = (_splitmix_np(5, 11, np.arange(m)) >= np.uint64(0x5555555555555556)).astype(np.int8)
    assert counts[s == 0].min() >= 1
    assert (s == 0).mean() == pytest.approx(1 / 3, abs=0.01)


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
