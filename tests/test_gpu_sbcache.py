"""GPU parity of the cluster shared-memory rank kernels (sbcache.cu) against the CPU oracle.

These kernels read the superblock words s_i / s_{i,c} from a
lossless re-encoding held in the shared memory of a 2-CTA cluster (6 superblocks per u64 for
BiRank16, 8 per u64 and symbol for QuadRank16).  The cases below put queries on every
superblock boundary of texts whose superblock counts straddle the group size (6 / 8) and the
CTA split (odd / even group counts), and use the texts that make the per-superblock increments
maximal (all-ones: +31 per BiRank superblock; a single repeated symbol: +7 per QuadRank
superblock), so every field of the encoding reaches its largest value.  Outputs must be
bit-identical to the oracle and to the global-memory kernels.
"""
import numpy as np
import pytest

import gen
import oracle
import paper_2602_04103_b200 as qr
from _util import B, B4, S, S4, boundary_queries, to_dev, to_host

pytestmark = pytest.mark.gpu

SB_COUNTS = [1, 2, 5, 6, 7, 11, 12, 13, 17, 24, 25, 61]


def _torch():
    import torch

    return torch


@pytest.fixture
def smem_mode():
    yield
    qr.qr_set_tuning("rank_smem", 1)
    qr.qr_set_tuning("rank_smem_k", 0)
    qr.qr_set_tuning("rank_dyn", 1)
    qr.qr_set_tuning("rank_smem_clusters", 0)


def _rank(h, q, c, dev, mode):
    torch = _torch()
    qr.qr_set_tuning("rank_smem", mode)
    dq = to_dev(q, dev)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, None if c is None else to_dev(c, dev), out)
    torch.cuda.synchronize()
    return to_host(out)


def _rank4(h, q, dev, mode):
    torch = _torch()
    qr.qr_set_tuning("rank_smem", mode)
    dq = to_dev(q, dev)
    out = torch.empty((q.size, 4), dtype=torch.uint64, device=dev)
    qr.qr_rank_all4(h, dq, out)
    torch.cuda.synchronize()
    return to_host(out)


def _bits(kind, n, seed):
    if kind == "ones":
        return np.full(max(1, (n + 63) // 64), np.uint64(0xFFFFFFFFFFFFFFFF))
    return gen.bits(seed, n, kind)


@pytest.mark.parametrize("k", SB_COUNTS)
@pytest.mark.parametrize("kind", [0.5, "ones", 0.01])
def test_birank_smem_parity(cuda, smem_mode, k, kind):
    for n in (k * S - 1, k * S, k * S + 1 + 977 * k):
        w = _bits(kind, n, 300 + k)
        h = qr.qr_birank_build(w, n)
        L = n // B + 1
        groups = ((L - 1) // 128 + 1 + 5) // 6
        assert qr.qr_super_cache_bytes(h) == 8 * (((groups + 1) // 2 + 1) & ~1)
        q = np.concatenate([boundary_queries(n, B, S, 240, limit=4000), gen.queries(11 + k, n, 50000)])
        ora = oracle.BitsOracle(w, n)
        got = _rank(h, q, None, cuda, 2)
        ref = ora.rank(q)
        bad = np.nonzero(got != ref)[0]
        assert bad.size == 0, f"n={n} {kind}: {bad.size} mismatches, q={q[bad[:4]]} got={got[bad[:4]]} ref={ref[bad[:4]]}"
        assert np.array_equal(got, _rank(h, q, None, cuda, 0))
        c = (gen.queries(5, 1, q.size, with_c=True)[1] & 1).astype(np.uint8)
        assert np.array_equal(_rank(h, q, c, cuda, 2), ora.rank(q, c))


@pytest.mark.parametrize("k", SB_COUNTS)
@pytest.mark.parametrize("kind", ["iid", "G", "T"])
def test_quadrank_smem_parity(cuda, smem_mode, k, kind):
    for n in (k * S4 - 1, k * S4 + 1 + 501 * k):
        if kind == "iid":
            t = gen.dna(400 + k, n)
        else:
            word = {"G": 0xAAAAAAAAAAAAAAAA, "T": 0xFFFFFFFFFFFFFFFF}[kind]
            t = np.full(max(1, (n + 31) // 32), np.uint64(word))
        h = qr.qr_quadrank_build(t, n)
        L = n // B4 + 1
        groups = ((L - 1) // 256 + 1 + 7) // 8
        assert qr.qr_super_cache_bytes(h) == 32 * ((groups + 1) // 2)
        q, c = gen.queries(21 + k, n, 40000, with_c=True)
        bq = boundary_queries(n, B4, S4, 96, limit=4000)
        q = np.concatenate([q, bq, bq, bq, bq])
        c = np.concatenate([c, np.repeat(np.arange(4, dtype=np.uint8), bq.size)])
        ora = oracle.DnaOracle(t, n)
        got = _rank(h, q, c, cuda, 2)
        ref = ora.rank(q, c)
        bad = np.nonzero(got != ref)[0]
        assert bad.size == 0, f"n={n} {kind}: {bad.size} mismatches, q={q[bad[:4]]} c={c[bad[:4]]}"
        assert np.array_equal(got, _rank(h, q, c, cuda, 0))
        g4 = _rank4(h, q, cuda, 2)
        assert np.array_equal(g4, ora.rank_all4(q))
        assert np.array_equal(g4, _rank4(h, q, cuda, 0))


@pytest.mark.parametrize("dyn", [0, 1])
@pytest.mark.parametrize("rank_k", [0, 1, 2, 4, 6, 8])
def test_smem_kernels_rank_k(cuda, smem_mode, rank_k, dyn):
    """Every (K, threads) instantiation of the cluster kernels, static and dynamic work order
    (results never depend on them)."""
    qr.qr_set_tuning("rank_smem_k", rank_k)
    qr.qr_set_tuning("rank_dyn", dyn)
    n = 9 * S + 4321
    w = gen.bits(77, n)
    q = np.concatenate([gen.queries(78, n, 123457), boundary_queries(n, B, S, 240)])
    h = qr.qr_birank_build(w, n)
    assert np.array_equal(_rank(h, q, None, cuda, 2), oracle.BitsOracle(w, n).rank(q))
    n4 = 13 * S4 + 99
    t = gen.dna(79, n4)
    q4, c4 = gen.queries(80, n4, 123457, with_c=True)
    h4 = qr.qr_quadrank_build(t, n4)
    ora4 = oracle.DnaOracle(t, n4)
    assert np.array_equal(_rank(h4, q4, c4, cuda, 2), ora4.rank(q4, c4))
    assert np.array_equal(_rank4(h4, q4, cuda, 2), ora4.rank_all4(q4))


def test_smem_auto_mode_large_batch_and_clone_import(cuda, smem_mode):
    """Default mode (1) takes the cluster path at m >= 2^22: checked on a 2^27-bit text, also on
    handles re-created by qr_import_layout and qr_clone_to_device (they rebuild the table)."""
    torch = _torch()
    n = (1 << 27) + 12345
    w = gen.bits(90, n)
    h = qr.qr_birank_build(w, n)
    m = (1 << 22) + 777
    q = gen.queries(91, n, m)
    ref = oracle.BitsOracle(w, n).rank(q)
    qr.qr_set_tuning("rank_smem", 1)
    dq = to_dev(q, cuda)
    lines, sup = qr.qr_export_layout(h)
    for hh in (h, qr.qr_import_layout(lines, sup, n, qr.QR_LAYOUT_BIRANK16), qr.qr_clone_to_device(h, 0)):
        assert qr.qr_super_cache_bytes(hh) > 0
        out = torch.empty_like(dq)
        qr.qr_rank(hh, dq, None, out)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(out), ref)


def test_no_cache_for_variants_and_fallback(cuda, smem_mode):
    """Layouts without an L1 array have no table; rank_smem = 2 then uses the global kernels."""
    n = 5 * S + 3
    w = gen.bits(93, n)
    hv = qr.qr_build(w, n, qr.QR_LAYOUT_BIRANK64X2)
    assert qr.qr_super_cache_bytes(hv) == 0
    q = gen.queries(94, n, 10000)
    assert np.array_equal(_rank(hv, q, None, cuda, 2), oracle.BitsOracle(w, n).rank(q))


def test_cache_capacity_limit(cuda, smem_mode):
    """The table is built iff half of it fits one CTA's opt-in shared memory (minus 1 KiB); at
    n = 2^34 (configs[1]) it must exist.  Beyond the limit rank still matches the oracle."""
    torch = _torch()
    optin = getattr(torch.cuda.get_device_properties(0), "shared_memory_per_block_optin", 232448)

    def expect(n):
        L = n // B + 1
        groups = ((L - 1) // 128 + 1 + 5) // 6
        half = 8 * (((groups + 1) // 2 + 1) & ~1)
        return half if half + 1024 <= optin else 0

    for n in ((1 << 34), (1 << 34) + (1 << 32)):
        bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=cuda)
        gen.bits_dev(95, n, 0.5, bits)
        h = qr.qr_birank_build(bits, n)
        del bits
        assert qr.qr_super_cache_bytes(h) == expect(n)
        if n == (1 << 34):
            assert expect(n) > 0
        m = 1 << 22
        q = torch.empty(m, dtype=torch.uint64, device=cuda)
        gen.queries_dev(96, n, m, q)
        out = torch.empty_like(q)
        qr.qr_set_tuning("rank_smem", 2)
        qr.qr_rank(h, q, None, out)
        qr.qr_set_tuning("rank_smem", 0)
        out0 = torch.empty_like(q)
        qr.qr_rank(h, q, None, out0)
        torch.cuda.synchronize()
        assert torch.equal(out, out0)
        h.free()
        del q, out, out0
        torch.cuda.empty_cache()


@pytest.mark.parametrize("clusters", [1, 3, 200])
def test_smem_cluster_count_does_not_change_results(cuda, smem_mode, clusters):
    """Fewer clusters than SMs (1, 3) or more than fit at once (200: a second wave) — both work
    orders must still cover every query exactly once."""
    qr.qr_set_tuning("rank_smem_clusters", clusters)
    n = 7 * S + 99
    w = gen.bits(81, n)
    q = gen.queries(82, n, 300001)
    h = qr.qr_birank_build(w, n)
    ref = oracle.BitsOracle(w, n).rank(q)
    for dyn in (0, 1):
        qr.qr_set_tuning("rank_dyn", dyn)
        assert np.array_equal(_rank(h, q, None, cuda, 2), ref)
    assert qr.qr_super_cache_clusters(h) > 0


def test_smem_concurrent_streams_and_staged_host_path(cuda, smem_mode):
    """The dynamic work order's counters are per launch (an event-guarded ring): launches of the
    cluster kernels on several streams at once, and the staged host-pointer path (chunks on the
    library's internal streams), all give the oracle's answers."""
    torch = _torch()
    qr.qr_set_tuning("rank_smem", 2)
    n = 11 * S + 321
    w = gen.bits(61, n)
    h = qr.qr_birank_build(w, n)
    q = gen.queries(62, n, 300000)
    ref = oracle.BitsOracle(w, n).rank(q)
    dq = to_dev(q, cuda)
    streams = [torch.cuda.Stream() for _ in range(6)]
    outs = [torch.empty_like(dq) for _ in streams]
    torch.cuda.synchronize()
    for rep in range(12):                      # more launches than streams: slots are reused
        for s, o in zip(streams, outs):
            with torch.cuda.stream(s):
                qr.qr_rank(h, dq, None, o, stream=s)
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(to_host(o), ref)
    qr.qr_set_tuning("stage_chunk", 65536)     # 5 chunks over the internal streams
    try:
        host_out = np.zeros(q.size, np.uint64)
        qr.qr_rank(h, q, None, host_out)
        qr.qr_sync()
        assert np.array_equal(host_out, ref)
        n4 = 5 * S4 + 77
        t = gen.dna(63, n4)
        h4 = qr.qr_quadrank_build(t, n4)
        q4, c4 = gen.queries(64, n4, 300000, with_c=True)
        o4 = np.zeros((q4.size, 4), np.uint64)
        qr.qr_rank_all4(h4, q4, o4)
        o1 = np.zeros(q4.size, np.uint64)
        qr.qr_rank(h4, q4, c4, o1)
        qr.qr_sync()
        ora4 = oracle.DnaOracle(t, n4)
        assert np.array_equal(o4, ora4.rank_all4(q4))
        assert np.array_equal(o1, ora4.rank(q4, c4))
    finally:
        qr.qr_set_tuning("stage_chunk", 1 << 23)


def test_smem_limit_never_lowered(cuda, smem_mode):
    """Regression: a launch with a small table must not lower the kernel's shared-memory limit
    below what an earlier (cached) larger table needs."""
    torch = _torch()
    qr.qr_set_tuning("rank_smem", 2)
    hs = []
    for n in ((1 << 32) + 5, 3 * S + 1, (1 << 32) + 5):
        bits = torch.empty((n + 63) // 64 + 1, dtype=torch.uint64, device=cuda)
        gen.bits_dev(70, n, 0.5, bits)
        h = qr.qr_birank_build(bits, n)
        m = 100000
        q = torch.empty(m, dtype=torch.uint64, device=cuda)
        gen.queries_dev(71, n, m, q)
        out = torch.empty_like(q)
        qr.qr_rank(h, q, None, out)
        qr.qr_set_tuning("rank_smem", 0)
        out0 = torch.empty_like(q)
        qr.qr_rank(h, q, None, out0)
        qr.qr_set_tuning("rank_smem", 2)
        torch.cuda.synchronize()
        assert torch.equal(out, out0)
        hs.append(h)


@pytest.mark.parametrize("dyn", [0, 1])
def test_global_kernels_dynamic_order_large_batch(cuda, smem_mode, dyn):
    """The global-memory lane-pair kernels (rank_smem = 0) and the layout variants take the
    dynamic work order for batches >= 2^22: every query answered once, bit-identical to the
    oracle; the gather ceilings load the same words in either order."""
    torch = _torch()
    qr.qr_set_tuning("rank_smem", 0)
    qr.qr_set_tuning("rank_dyn", dyn)
    m = (1 << 22) + 999
    n = 21 * S + 5
    w = gen.bits(110, n)
    q = gen.queries(111, n, m)
    ora = oracle.BitsOracle(w, n)
    ref = ora.rank(q)
    dq = to_dev(q, cuda)
    c = (gen.queries(112, 1, m, with_c=True)[1] & 1).astype(np.uint8)
    for layout in (qr.QR_LAYOUT_BIRANK16, qr.QR_LAYOUT_BIRANK64X2):
        h = qr.qr_build(w, n, layout)
        out = torch.empty_like(dq)
        qr.qr_rank(h, dq, None, out)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(out), ref), layout
        qr.qr_rank(h, dq, to_dev(c, cuda), out)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(out), ora.rank(q, c)), layout
        g = {}
        for d in (0, 1):
            qr.qr_set_tuning("rank_dyn", d)
            qr.qr_gather_ceiling(h, dq, out, 0)
            torch.cuda.synchronize()
            g[d] = to_host(out).copy()
        qr.qr_set_tuning("rank_dyn", dyn)
        assert np.array_equal(g[0], g[1]), layout
    n4 = 9 * S4 + 3
    t = gen.dna(113, n4)
    q4, c4 = gen.queries(114, n4, m, with_c=True)
    ora4 = oracle.DnaOracle(t, n4)
    dq4 = to_dev(q4, cuda)
    for layout in (qr.QR_LAYOUT_QUADRANK16, qr.QR_LAYOUT_QUADRANK64):
        h4 = qr.qr_build(t, n4, layout)
        o = torch.empty_like(dq4)
        qr.qr_rank(h4, dq4, to_dev(c4, cuda), o)
        o4 = torch.empty((m, 4), dtype=torch.uint64, device=cuda)
        qr.qr_rank_all4(h4, dq4, o4)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(o), ora4.rank(q4, c4)), layout
        assert np.array_equal(to_host(o4), ora4.rank_all4(q4)), layout


@pytest.mark.parametrize("lane_table", [0, 1])
@pytest.mark.parametrize("m", [100003, (1 << 22) + 5])
def test_lane_kernels_l2_resident(cuda, smem_mode, lane_table, m):
    """L2-resident structures take one lane per query (rank_shape LANE): superblock words from a
    per-CTA shared-memory copy of the packed table (rank_lane_table 1, default) or from L2 (0);
    static (m < 2^22) and dynamic order; rank, rank with c, QuadRank rank and rank_4."""
    qr.qr_set_tuning("rank_lane_table", lane_table)
    try:
        n = 37 * S + 1234
        w = gen.bits(120, n, 1.0 if m < 200000 else 0.5)
        q = gen.queries(121, n, m)
        h = qr.qr_birank_build(w, n)
        ora = oracle.BitsOracle(w, n)
        got = _rank(h, q, None, cuda, 1)
        assert np.array_equal(got, ora.rank(q))
        c = (gen.queries(122, 1, m, with_c=True)[1] & 1).astype(np.uint8)
        assert np.array_equal(_rank(h, q, c, cuda, 1), ora.rank(q, c))
        n4 = 29 * S4 + 77
        t = gen.dna(123, n4)
        q4, c4 = gen.queries(124, n4, m, with_c=True)
        h4 = qr.qr_quadrank_build(t, n4)
        ora4 = oracle.DnaOracle(t, n4)
        assert np.array_equal(_rank(h4, q4, c4, cuda, 1), ora4.rank(q4, c4))
        assert np.array_equal(_rank4(h4, q4, cuda, 1), ora4.rank_all4(q4))
    finally:
        qr.qr_set_tuning("rank_lane_table", 1)


def test_cuda_graph_capture_of_dynamic_order_launches(cuda, smem_mode):
    """qr_rank (cluster kernel, dynamic order: m >= 2^22), qr_rank_all4 and qr_fm_count captured
    into CUDA graphs and replayed: the work counters become graph-owned allocations during a
    capture, so replays give the oracle's answers."""
    torch = _torch()
    n = (1 << 27) + 99
    w = gen.bits(130, n)
    h = qr.qr_birank_build(w, n)
    m = (1 << 22) + 3
    q = gen.queries(131, n, m)
    ref = oracle.BitsOracle(w, n).rank(q)
    dq = to_dev(q, cuda)
    out = torch.zeros_like(dq)
    s = torch.cuda.Stream()
    qr.qr_rank(h, dq, None, out, stream=s)            # warm-up outside the capture (one-time setup)
    torch.cuda.synchronize()
    for mode in (2, 1):                               # cluster kernel, then the size-chosen shape
        qr.qr_set_tuning("rank_smem", mode)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            qr.qr_rank(h, dq, None, out, stream=torch.cuda.current_stream())
        for _ in range(3):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert np.array_equal(to_host(out), ref), mode
    n4 = 7 * S4 + 5
    t = gen.dna(132, n4)
    h4 = qr.qr_quadrank_build(t, n4)
    q4 = gen.queries(133, n4, m)
    dq4 = to_dev(q4, cuda)
    o4 = torch.zeros((m, 4), dtype=torch.uint64, device=cuda)
    qr.qr_rank_all4(h4, dq4, o4, stream=s)
    torch.cuda.synchronize()
    g4 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g4, stream=s):
        qr.qr_rank_all4(h4, dq4, o4, stream=torch.cuda.current_stream())
    o4.zero_()
    g4.replay()
    torch.cuda.synchronize()
    assert np.array_equal(to_host(o4), oracle.DnaOracle(t, n4).rank_all4(q4))
    nf = 200000
    tf = gen.dna(134, nf)
    fm = qr.qr_fm_build(tf, nf)
    L, mp = 24, 5000
    pats = gen.patterns(135, 0, mp, L, tf, nf)
    dp = to_dev(pats, cuda)
    d = torch.zeros(mp, dtype=torch.int32, device=cuda)
    qr.qr_fm_count(fm, dp, None, L, d, mp, stream=s)
    torch.cuda.synchronize()
    gf = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf, stream=s):
        qr.qr_fm_count(fm, dp, None, L, d, mp, stream=torch.cuda.current_stream())
    d.zero_()
    gf.replay()
    torch.cuda.synchronize()
    ref_fm = oracle.FmOracle(gen.unpack_dna(tf, nf)).count(pats, np.arange(mp, dtype=np.uint64) * L,
                                                          np.full(mp, L, np.uint32))
    assert np.array_equal(to_host(d).view(np.uint32), ref_fm)
    # approximate counting (k = 1, 2) and both strands, captured the same way
    sym = gen.unpack_dna(tf, nf)
    offs, lens = np.arange(mp, dtype=np.uint64) * L, np.full(mp, L, np.uint32)
    for k in (1, 2):
        da = torch.zeros(mp, dtype=torch.int32, device=cuda)
        qr.qr_fm_count_approx(fm, dp, None, L, k, da, mp, stream=s)
        torch.cuda.synchronize()
        ga = torch.cuda.CUDAGraph()
        with torch.cuda.graph(ga, stream=s):
            qr.qr_fm_count_approx(fm, dp, None, L, k, da, mp, stream=torch.cuda.current_stream())
        da.zero_()
        ga.replay()
        torch.cuda.synchronize()
        assert np.array_equal(to_host(da).view(np.uint32), oracle.scan_count_hdk(sym, pats, offs, lens, k)), k
    df, dr = torch.zeros(mp, dtype=torch.int32, device=cuda), torch.zeros(mp, dtype=torch.int32, device=cuda)
    qr.qr_fm_count_both(fm, dp, None, L, df, dr, mp, stream=s)
    torch.cuda.synchronize()
    gb = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gb, stream=s):
        qr.qr_fm_count_both(fm, dp, None, L, df, dr, mp, stream=torch.cuda.current_stream())
    df.zero_(); dr.zero_()
    gb.replay()
    torch.cuda.synchronize()
    rc = np.concatenate([3 - pats[i * L:(i + 1) * L][::-1] for i in range(mp)]).astype(np.uint8)
    assert np.array_equal(to_host(df).view(np.uint32), ref_fm)
    assert np.array_equal(to_host(dr).view(np.uint32), oracle.FmOracle(sym).count(rc, offs, lens))


@pytest.mark.parametrize("resident", [1, 0])
@pytest.mark.parametrize("nb,n4", [(1, 1), (1000, 700), (1 << 20, 1 << 19), (1_400_000, 600_000), (3_000_000, 1_000_000)])
def test_resident_structure_parity(cuda, smem_mode, resident, nb, n4):
    """Structures small enough for one CTA's shared memory (configs[0]-sized and up to the
    200 KB limit; the last size does not fit and takes the L2 path) queried from the per-CTA copy
    (rank_resident 1) or from L2 (0): rank, rank with c, QuadRank rank and rank_4 on batches large
    enough for the resident path, boundary queries included."""
    qr.qr_set_tuning("rank_resident", resident)
    try:
        # the resident path needs 16 B/query >= 2x (148 copies of the structure): 3.5M queries
        # cover the largest structures that fit
        m = 3_500_000 if nb >= (1 << 20) else 300000
        w = gen.bits(140 + nb % 7, nb)
        q = np.concatenate([gen.queries(141, nb, m), boundary_queries(nb, B, S, 240, limit=5000)])
        h = qr.qr_birank_build(w, nb)
        ora = oracle.BitsOracle(w, nb)
        assert np.array_equal(_rank(h, q, None, cuda, 1), ora.rank(q))
        c = (gen.queries(142, 1, q.size, with_c=True)[1] & 1).astype(np.uint8)
        assert np.array_equal(_rank(h, q, c, cuda, 1), ora.rank(q, c))
        t = gen.dna(143 + n4 % 5, n4)
        m = 3_500_000 if n4 >= (1 << 19) else 300000
        q4, c4 = gen.queries(144, n4, m, with_c=True)
        bq = boundary_queries(n4, B4, S4, 96, limit=5000)
        q4 = np.concatenate([q4, bq]); c4 = np.concatenate([c4, (bq % 4).astype(np.uint8)])
        h4 = qr.qr_quadrank_build(t, n4)
        ora4 = oracle.DnaOracle(t, n4)
        assert np.array_equal(_rank(h4, q4, c4, cuda, 1), ora4.rank(q4, c4))
        assert np.array_equal(_rank4(h4, q4, cuda, 1), ora4.rank_all4(q4))
    finally:
        qr.qr_set_tuning("rank_resident", 1)


def test_large_table_limit_large_small_large(cuda, smem_mode):
    """Regression: the CS-CTA cluster launcher cached its grid per (kernel, table size)
    and set the shared-memory limit only on a cache miss, so large -> small -> large handle order
    launched the large table above a lowered limit (QR_ECUDA).  Tables of ~180 KB (2^35 bits) and
    ~111 KB (1.23 x 2^34 bits, forced onto the large-n table) per CTA, queried in that order; every
    result equals the global-memory kernel's."""
    torch = _torch()
    qr.qr_set_tuning("rank_big_pack", 1)
    hs = {}
    try:
        for key, n in (("A", 1 << 35), ("B", int(1.23 * (1 << 34)))):
            bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=cuda)
            gen.bits_dev(72, n, 0.5, bits)
            hs[key] = (qr.qr_birank_build(bits, n), n)
            del bits
    finally:
        qr.qr_set_tuning("rank_big_pack", 0)
    m = (1 << 22) + 5
    for key in ("A", "B", "A"):
        h, n = hs[key]
        q = torch.empty(m, dtype=torch.uint64, device=cuda)
        gen.queries_dev(73, n, m, q)
        out = torch.empty_like(q)
        qr.qr_set_tuning("rank_smem", 1)
        qr.qr_rank(h, q, None, out)
        qr.qr_set_tuning("rank_smem", 0)
        ref = torch.empty_like(q)
        qr.qr_rank(h, q, None, ref)
        qr.qr_set_tuning("rank_smem", 1)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), key


def test_import_layout_rejects_wrong_sizes(cuda, smem_mode):
    """qr_import_layout checks the buffers' byte counts against (n, layout) before copying."""
    n = 5 * S + 3
    w = gen.bits(94, n)
    h = qr.qr_birank_build(w, n)
    lines, sup = qr.qr_export_layout(h)
    with pytest.raises(qr.QrError, match="differ"):
        qr.qr_import_layout(lines[:-64], sup, n, qr.QR_LAYOUT_BIRANK16)
    with pytest.raises(qr.QrError, match="differ"):
        qr.qr_import_layout(lines, sup, n + S, qr.QR_LAYOUT_BIRANK16)
    with pytest.raises(qr.QrError):
        qr.qr_import_layout(lines, None, n, qr.QR_LAYOUT_BIRANK16)
    h2 = qr.qr_import_layout(lines, sup, n, qr.QR_LAYOUT_BIRANK16)
    q = gen.queries(95, n, 5000)
    assert np.array_equal(_rank(h2, q, None, cuda, 0), oracle.BitsOracle(w, n).rank(q))


@pytest.mark.parametrize("cs", [4, 8, 16])
@pytest.mark.parametrize("n_sb,extra", [(1, 5), (37, 1234), (401, 77)])
def test_large_table_cluster_kernel_parity(cuda, smem_mode, cs, n_sb, extra):
    """The BiRank16 table for n >= 2^35 (5-superblock groups with a 32-bit base over a 4/8/16-CTA
    cluster), forced onto small n: rank and rank with c on >= 2^22 queries + the boundary set."""
    qr.qr_set_tuning("rank_big_pack", 1)
    qr.qr_set_tuning("rank_big_cs", cs)
    try:
        n = n_sb * S + extra
        w = gen.bits(800 + n_sb, n)
        h = qr.qr_birank_build(w, n)
    finally:
        qr.qr_set_tuning("rank_big_pack", 0)
        qr.qr_set_tuning("rank_big_cs", 0)
    m = (1 << 22) + 11
    q = np.concatenate([gen.queries(801, n, m), boundary_queries(n, B, S, 240, limit=20000)])
    ora = oracle.BitsOracle(w, n)
    assert np.array_equal(_rank(h, q, None, cuda, 1), ora.rank(q))
    c = (gen.queries(802, 1, q.size, with_c=True)[1] & 1).astype(np.uint8)
    assert np.array_equal(_rank(h, q, c, cuda, 1), ora.rank(q, c))


@pytest.mark.parametrize("cs", [4, 8, 16])
@pytest.mark.parametrize("n_sb,extra", [(1, 3), (23, 777), (300, 5)])
def test_large_table_cluster_kernel_quadrank(cuda, smem_mode, cs, n_sb, extra):
    """QuadRank16's 8-superblock groups over a 4/8/16-CTA cluster (n > ~2^32.6 chars), forced
    onto small n: rank(q, c) and rank_4 on >= 2^22 queries + the boundary set."""
    qr.qr_set_tuning("rank_big_pack", 1)
    qr.qr_set_tuning("rank_big_cs", cs)
    try:
        n = n_sb * S4 + extra
        t = gen.dna(900 + n_sb, n)
        h = qr.qr_quadrank_build(t, n)
    finally:
        qr.qr_set_tuning("rank_big_pack", 0)
        qr.qr_set_tuning("rank_big_cs", 0)
    m = (1 << 22) + 7
    q, c = gen.queries(901, n, m, with_c=True)
    bq = boundary_queries(n, B4, S4, 96, limit=20000)
    q = np.concatenate([q, bq]); c = np.concatenate([c, (bq % 4).astype(np.uint8)])
    ora = oracle.DnaOracle(t, n)
    assert np.array_equal(_rank(h, q, c, cuda, 1), ora.rank(q, c))
    assert np.array_equal(_rank4(h, q, cuda, 1), ora.rank_all4(q))
