"""GPU parity of the bucketed BiRank16 rank path (bucket.cu) against the CPU oracle.

Large batches over structures much larger than the L2 are answered by regrouping the queries
by line region (histogram, scatter, Eq. 1 per entry with the line from the L2, unpermute);
every query is still Eq. 1 on its own line, so every output must equal the
oracle's rank(q) = sum_{i<q} t_i, and with c the sigma = 2 convention
c ? rank1 : q - rank1.  The path is forced on small texts here
(rank_bucket = 2): the automatic bucket shift then gives hundreds of buckets of a few lines,
and the forced destination shift hundreds of output groups, so tiles straddle buckets and
groups, buckets are empty or hold every query, and tiles are ragged.
"""
import numpy as np
import pytest

import gen
import oracle
import paper_2602_04103_b200 as qr
from _util import B, S, boundary_queries, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture
def bucket():
    qr.qr_set_tuning("rank_bucket", 2)
    yield
    qr.qr_set_tuning("rank_bucket", 1)
    qr.qr_set_tuning("rank_bucket_shift", 0)
    qr.qr_set_tuning("rank_bucket_dshift", 0)
    qr.qr_set_tuning("rank_bucket_chunk", 1 << 31)


def _run(h, q, c, dev, inplace=False):
    import torch

    dq = to_dev(q, dev)
    dc = None if c is None else to_dev(c, dev)
    out = dq if inplace else torch.empty_like(dq)
    qr.qr_rank(h, dq, dc, out)
    torch.cuda.synchronize()
    return to_host(out)


def _expect(orc, q, c):
    r = orc.rank(q)
    if c is None:
        return r
    return np.where(c != 0, r, q - r).astype(np.uint64)


def _queries(kind, n, m, seed):
    if kind == "uniform":
        return gen.queries(seed, n, m)
    if kind == "one":                       # every query in one bucket (and one line)
        return np.full(m, n // 3, np.uint64)
    if kind == "sorted":
        return np.sort(gen.queries(seed, n, m))
    if kind == "reverse":
        return np.sort(gen.queries(seed, n, m))[::-1].copy()
    if kind == "ends":                      # only the first and the last bucket
        q = gen.queries(seed, min(n, 3 * B), m)
        q[1::2] = n - q[1::2] % min(n + 1, 3 * B)
        return q
    raise ValueError(kind)


@pytest.mark.parametrize("n", [1, B - 1, 3 * S + 5, 1_000_003, 7_777_777])
@pytest.mark.parametrize("kind", ["uniform", "one", "sorted", "reverse", "ends"])
def test_bucket_rank_vs_oracle(cuda, bucket, n, kind):
    w = gen.bits(31, n)
    h = qr.qr_birank_build(w, n)
    orc = oracle.BitsOracle(w, n)
    for m in (1, 8191, 8192, 8193, 100_003):
        q = _queries(kind, n, m, 7 + m)
        assert np.array_equal(_run(h, q, None, cuda), _expect(orc, q, None)), (n, kind, m)


@pytest.mark.parametrize("dshift", [0, 6, 13])
def test_bucket_rank_with_c_and_groups(cuda, bucket, dshift):
    n = 2_000_017
    w = gen.bits(32, n, p=0.01)
    h = qr.qr_birank_build(w, n)
    orc = oracle.BitsOracle(w, n)
    qr.qr_set_tuning("rank_bucket_dshift", dshift)
    m = 300_001
    q = np.concatenate([boundary_queries(n, B, S, 240), gen.queries(3, n, m)])
    c = (gen.queries(4, 1, q.size) & 1).astype(np.uint8)
    assert np.array_equal(_run(h, q, c, cuda), _expect(orc, q, c))
    assert np.array_equal(_run(h, q, None, cuda), _expect(orc, q, None))


@pytest.mark.parametrize("shift", [0, 3, 9])
def test_bucket_shift_and_chunks(cuda, bucket, shift):
    """Forced bucket widths (few wide buckets) and batches split into chunks of 2^k queries."""
    n = 5_000_011
    w = gen.bits(33, n)
    h = qr.qr_birank_build(w, n)
    orc = oracle.BitsOracle(w, n)
    qr.qr_set_tuning("rank_bucket_shift", shift)
    q = gen.queries(5, n, 250_000)
    c = (gen.queries(6, 1, q.size) & 1).astype(np.uint8)
    exp = _expect(orc, q, c)
    assert np.array_equal(_run(h, q, c, cuda), exp)
    for chunk in (8192, 65_537):
        qr.qr_set_tuning("rank_bucket_chunk", chunk)
        assert np.array_equal(_run(h, q, c, cuda), exp), chunk


def test_bucket_inplace_and_contract(cuda, bucket):
    """out == q (the scatter then takes a buffer of its own); q > n must not fault."""
    n = 3_000_001
    w = gen.bits(34, n)
    h = qr.qr_birank_build(w, n)
    orc = oracle.BitsOracle(w, n)
    q = gen.queries(8, n, 200_000)
    assert np.array_equal(_run(h, q, None, cuda, inplace=True), orc.rank(q))
    big = np.array([n + 1, n + 496, 2 * n, 1 << 40, (1 << 64) - 1] * 3000, np.uint64)
    _run(h, big, None, cuda)
    qr.qr_sync()


def test_bucket_matches_direct_default_path(cuda):
    """The automatic choice: identical outputs with the bucketed path on and off."""
    n = 9_000_001
    w = gen.bits(35, n)
    h = qr.qr_birank_build(w, n)
    q = gen.queries(9, n, 1 << 20)
    try:
        qr.qr_set_tuning("rank_bucket", 0)
        a = _run(h, q, None, cuda)
        qr.qr_set_tuning("rank_bucket", 2)
        b = _run(h, q, None, cuda)
    finally:
        qr.qr_set_tuning("rank_bucket", 1)
    assert np.array_equal(a, b)
    assert np.array_equal(a, oracle.BitsOracle(w, n).rank(q))
