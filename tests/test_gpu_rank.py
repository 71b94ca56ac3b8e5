"""GPU parity of BiRank16 / QuadRank16 (rank, rank_all4, layout) against the CPU oracle.

Every comparison is element-by-element and bit-exact (integer outputs), on seeded
inputs from gen/, at sizes that span several lines and superblocks with ragged
tails, plus the degenerate cases (n = 0, 1, B-1, B, B+1, all-zero, all-one, all-G).
"""
import numpy as np
import pytest

import gen
import oracle
import paper_2602_04103_b200 as qr
from _util import B, B4, S, S4, boundary_queries, to_dev, to_host

pytestmark = pytest.mark.gpu

BI_SIZES = [0, 1, 2, 63, 64, 240, 241, 495, 496, 497, 991, 992, 993, S - 1, S, S + 1, 2 * S + 7, 5 * S + 4321,
            (1 << 20)]
QD_SIZES = [0, 1, 31, 32, 95, 96, 97, 223, 224, 225, 447, 448, S4 - 1, S4, S4 + 1, 3 * S4 + 12345, (1 << 20) + 17]


def _torch():
    import torch

    return torch


def bits_for(n, p, seed):
    if p == "zeros":
        return np.zeros(max(1, (n + 63) // 64), np.uint64)
    return gen.bits(seed, n, p)


# ------------------------------------------------------------------ BiRank
@pytest.mark.parametrize("n", BI_SIZES)
@pytest.mark.parametrize("p", [0.5, 0.01, 1.0, "zeros"])
def test_birank_rank_parity(cuda, n, p):
    torch = _torch()
    w = bits_for(n, p, 1000 + n)
    ora = oracle.BitsOracle(w, n)
    h = qr.qr_birank_build(w, n, device=0)                       # host input pointer
    if n <= 200000:
        q = np.arange(n + 1, dtype=np.uint64)
    else:
        q = np.concatenate([gen.queries(7, n, 300000), boundary_queries(n, B, S, 240)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, out)
    torch.cuda.synchronize()
    got = to_host(out)
    ref = ora.rank(q)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"n={n} p={p}: {bad.size} mismatches, first q={q[bad[:5]]} got={got[bad[:5]]} ref={ref[bad[:5]]}"
    # sigma = 2 with a symbol array: c = 0 -> q - rank(q)
    c = (gen.queries(3, 1, q.size, with_c=True)[1] & 1).astype(np.uint8)
    out2 = torch.empty_like(dq)
    qr.qr_rank(h, dq, to_dev(c, cuda), out2)
    assert np.array_equal(to_host(out2), ora.rank(q, c))


def test_birank_layout_closed_forms(cuda):
    """Decode every line: b_j = rank(jB+240) - 2^11 s_{j>>7}, s_i = rank(iS)>>11 (:407),
    data bits = text; all-ones b_0 = 240 (golden); byte accounting = 3.2762%."""
    for n, p in [(5 * S + 4321, 0.5), (3 * S + 17, 1.0), (1000, 0.01)]:
        w = gen.bits(55, n, p)
        h = qr.qr_birank_build(w, n)
        lines, sup = qr.qr_export_layout(h)
        L = n // B + 1
        assert lines.size == 64 * L and sup.size == (L - 1) // 128 + 1
        u16 = lines.view(np.uint16).reshape(L, 32)
        ora = oracle.BitsOracle(w, n)
        anchors = np.minimum(np.arange(L, dtype=np.uint64) * B + 240, n)
        b = u16[:, 0].astype(np.uint64) + (sup[np.arange(L) // 128].astype(np.uint64) << 11)
        assert np.array_equal(b, ora.rank(anchors))
        sb = np.minimum(np.arange(sup.size, dtype=np.uint64) * S, n)
        assert np.array_equal(sup.astype(np.uint64), ora.rank(sb) >> 11)
        text16 = np.zeros(31 * L, np.uint16)
        t = w.view(np.uint16)[: min(w.size * 4, 31 * L)]
        text16[: t.size] = t
        assert np.array_equal(u16[:, 1:].reshape(-1), text16)
        if p == 1.0:
            assert u16[0, 0] == 240
    n = 1 << 24
    h = qr.qr_birank_build(gen.bits(1, n), n)
    overhead = (h.line_bytes + h.super_bytes) / (n / 8) - 1
    assert abs(overhead - (16 / 496 + 32 / S)) < 2e-4
    assert abs(round(overhead * 100, 2) - 3.28) < 0.011


def test_birank_device_input_and_host_query_path(cuda):
    torch = _torch()
    n = 3 * S + 999
    w = gen.bits(9, n)
    h = qr.qr_birank_build(to_dev(w, cuda), n)                   # device input pointer
    q = gen.queries(4, n, 100000)
    ref = oracle.BitsOracle(w, n).rank(q)
    out_h = np.zeros(q.size, np.uint64)
    qr.qr_set_tuning("stage_chunk", 4096)                        # many chunks through both slots
    try:
        qr.qr_rank(h, q, None, out_h)                            # host pointers: staged path
        qr.qr_sync()
    finally:
        qr.qr_set_tuning("stage_chunk", 1 << 23)
    assert np.array_equal(out_h, ref)
    qp = torch.from_numpy(q).pin_memory()
    op = torch.zeros_like(qp).pin_memory()
    qr.qr_rank(h, qp, None, op)
    torch.cuda.synchronize()
    assert np.array_equal(op.numpy(), ref)


@pytest.mark.parametrize("pair", [0, 1, 2])
@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_birank_tuning_does_not_change_results(cuda, k, pair):
    torch = _torch()
    n = 7 * S + 5
    w = gen.bits(17, n)
    h = qr.qr_birank_build(w, n)
    q = np.concatenate([gen.queries(5, n, 200001), boundary_queries(n, B, S, 240)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    c = (gen.queries(3, 1, q.size, with_c=True)[1] & 1).astype(np.uint8)
    out2 = torch.empty_like(dq)
    qr.qr_set_tuning("rank_k", k)
    qr.qr_set_tuning("rank_blocks_per_sm", 1 + k)
    qr.qr_set_tuning("rank_pair", pair)
    try:
        qr.qr_rank(h, dq, None, out)
        qr.qr_rank(h, dq, to_dev(c, cuda), out2)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("rank_k", 2)
        qr.qr_set_tuning("rank_blocks_per_sm", 64)
        qr.qr_set_tuning("rank_pair", 2)
    ora = oracle.BitsOracle(w, n)
    assert np.array_equal(to_host(out), ora.rank(q))
    assert np.array_equal(to_host(out2), ora.rank(q, c))


@pytest.mark.parametrize("pair", [0, 1, 2])
@pytest.mark.parametrize("k", [1, 2, 8])
def test_quadrank_tuning_does_not_change_results(cuda, k, pair):
    torch = _torch()
    n = 3 * S4 + 777
    w = gen.dna(19, n)
    h = qr.qr_quadrank_build(w, n)
    q, c = gen.queries(5, n, 100001, with_c=True)
    q = np.concatenate([q, boundary_queries(n, B4, S4, 96)])
    c = np.concatenate([c, (np.arange(q.size - c.size) % 4).astype(np.uint8)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    o4 = torch.empty((q.size, 4), dtype=torch.uint64, device=cuda)
    g = torch.empty_like(dq)
    qr.qr_set_tuning("rank_k", k)
    qr.qr_set_tuning("rank_blocks_per_sm", 2 + k)
    qr.qr_set_tuning("rank_pair", pair)
    try:
        qr.qr_rank(h, dq, to_dev(c, cuda), out)
        qr.qr_rank_all4(h, dq, o4)
        qr.qr_gather_ceiling(h, dq, g, 1)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("rank_k", 2)
        qr.qr_set_tuning("rank_blocks_per_sm", 64)
        qr.qr_set_tuning("rank_pair", 2)
    ora = oracle.DnaOracle(w, n)
    assert np.array_equal(to_host(out), ora.rank(q, c))
    assert np.array_equal(to_host(o4), ora.rank_all4(q))
    lines, _ = qr.qr_export_layout(h)
    u64 = lines.view(np.uint64).reshape(-1, 8)
    assert np.array_equal(to_host(g), np.bitwise_xor.reduce(u64[(q // B4).astype(np.int64)], axis=1))


@pytest.mark.parametrize("pair", [0, 1, 2])
def test_gather_ceiling_loads_the_same_sectors(cuda, pair):
    torch = _torch()
    qr.qr_set_tuning("rank_pair", pair)
    n = 4 * S + 77
    w = gen.bits(3, n)
    h = qr.qr_birank_build(w, n)
    lines, _ = qr.qr_export_layout(h)
    u64 = lines.view(np.uint64).reshape(-1, 8)
    q = gen.queries(8, n, 50000)
    dq = to_dev(q, cuda)
    for mode in (0, 1):
        out = torch.empty_like(dq)
        qr.qr_gather_ceiling(h, dq, out, mode)
        torch.cuda.synchronize()
        j = (q // B).astype(np.int64)
        p = 16 + q - j.astype(np.uint64) * B
        a = np.bitwise_xor.reduce(u64[j, :4], axis=1)
        b = np.bitwise_xor.reduce(u64[j, 4:], axis=1)
        exp = a ^ np.where((p >= 256) | (mode == 1), b, 0).astype(np.uint64)
        assert np.array_equal(to_host(out), exp)
    qr.qr_set_tuning("rank_pair", 2)


# ------------------------------------------------------------------ QuadRank
@pytest.mark.parametrize("n", QD_SIZES)
def test_quadrank_rank_and_all4_parity(cuda, n):
    torch = _torch()
    w = gen.dna(2000 + n, n)
    ora = oracle.DnaOracle(w, n)
    h = qr.qr_quadrank_build(w, n)
    if n <= 60000:
        q = np.repeat(np.arange(n + 1, dtype=np.uint64), 4)
        c = np.tile(np.arange(4, dtype=np.uint8), n + 1)
    else:
        q = np.concatenate([gen.queries(7, n, 300000), boundary_queries(n, B4, S4, 96)])
        c = (gen.queries(9, n, q.size, with_c=True)[1]).astype(np.uint8)
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, to_dev(c, cuda), out)
    torch.cuda.synchronize()
    got, ref = to_host(out), ora.rank(q, c)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"n={n}: {bad.size} mismatches, q={q[bad[:5]]} c={c[bad[:5]]} got={got[bad[:5]]} ref={ref[bad[:5]]}"
    qu = np.unique(q)
    out4 = torch.empty((qu.size, 4), dtype=torch.uint64, device=cuda)
    qr.qr_rank_all4(h, to_dev(qu, cuda), out4)
    torch.cuda.synchronize()
    a4 = to_host(out4)
    assert np.array_equal(a4, ora.rank_all4(qu))
    assert np.array_equal(a4.sum(axis=1), qu)                    # sum_c rank(q,c) = q


def test_quadrank_all_G_and_layout(cuda):
    """all-G deltas (0,0,96,0) (golden); b_{j,c}, s_{i,c} closed forms;
    plane soundness: (w_low ^ cl) & (w_high ^ ch) marks exactly the chars equal to c; 14.40%."""
    n = 3 * S4 + 1000
    w = np.full((n + 31) // 32, 0xAAAAAAAAAAAAAAAA, np.uint64)
    h = qr.qr_quadrank_build(w, n)
    lines, sup = qr.qr_export_layout(h)
    u16 = lines.view(np.uint16).reshape(-1, 32)
    assert list(u16[0, [0, 1, 4, 5]]) == [0, 0, 96, 0]
    for n, seed in [(3 * S4 + 12345, 4), (5000, 5)]:
        w = gen.dna(seed, n)
        h = qr.qr_quadrank_build(w, n)
        lines, sup = qr.qr_export_layout(h)
        L = n // B4 + 1
        u16 = lines.view(np.uint16).reshape(L, 32)
        u64 = lines.view(np.uint64).reshape(L, 8)
        sup = sup.reshape(-1, 4).astype(np.uint64)
        ora = oracle.DnaOracle(w, n)
        anchors = np.minimum(np.arange(L, dtype=np.uint64) * B4 + 96, n)
        for c, slot in enumerate([0, 1, 4, 5]):
            b = u16[:, slot].astype(np.uint64) + (sup[np.arange(L) // 256, c] << 13)
            # beyond n the padding is A: rank(x, A) grows past n, other symbols stay
            extra = np.zeros(L, np.uint64)
            if c == 0:
                extra = (np.arange(L, dtype=np.uint64) * B4 + 96) - anchors
            assert np.array_equal(b, ora.rank(anchors, np.full(L, c, np.uint8)) + extra), c
        sym = gen.unpack_dna(w, n)
        pad = np.zeros(L * B4, np.uint8)
        pad[:n] = sym
        pad = pad.reshape(L, B4)
        for c in range(4):
            cl = np.uint64(0xFFFFFFFFFFFFFFFF if c & 1 else 0)
            ch = np.uint64(0xFFFFFFFFFFFFFFFF if c >> 1 else 0)
            match = [(u64[:, 4 * hh + 2 * t] ^ cl) & (u64[:, 4 * hh + 2 * t + 1] ^ ch) for hh in (0, 1) for t in (0, 1)]
            bits = np.unpackbits(np.stack(match, axis=1).view(np.uint8), bitorder="little").reshape(L, 256)
            assert np.array_equal(bits[:, 32:].astype(bool), pad == c), c
    n = 1 << 24
    h = qr.qr_quadrank_build(gen.dna(1, n), n)
    overhead = (h.line_bytes + h.super_bytes) / (n / 4) - 1
    assert abs(round(overhead * 100, 2) - 14.40) < 0.011


def test_quadrank_host_path_and_c_mod4(cuda):
    n = 2 * S4 + 3
    w = gen.dna(12, n)
    h = qr.qr_quadrank_build(to_dev(w, cuda), n)
    q, c = gen.queries(6, n, 70000, with_c=True)
    ora = oracle.DnaOracle(w, n)
    out = np.zeros(q.size, np.uint64)
    qr.qr_set_tuning("stage_chunk", 8192)
    try:
        qr.qr_rank(h, q, (c | 4).astype(np.uint8), out)          # symbols are taken mod 4
        out4 = np.zeros((q.size, 4), np.uint64)
        qr.qr_rank_all4(h, q, out4)
        qr.qr_sync()
    finally:
        qr.qr_set_tuning("stage_chunk", 1 << 23)
    assert np.array_equal(out, ora.rank(q, c))
    assert np.array_equal(out4, ora.rank_all4(q))


def test_errors_surface(cuda):
    torch = _torch()
    n = 1000
    hb = qr.qr_birank_build(gen.bits(1, n), n)
    q = torch.zeros(10, dtype=torch.uint64, device=cuda)
    o4 = torch.zeros(40, dtype=torch.uint64, device=cuda)
    with pytest.raises(qr.QrError) as e:
        qr.qr_rank_all4(hb, q, o4)
    assert e.value.status == qr.QR_EINVAL
    hq = qr.qr_quadrank_build(gen.dna(1, n), n)
    with pytest.raises(qr.QrError):
        qr.qr_rank(hq, q, None, o4[:10])                        # sigma=4 needs c
    with pytest.raises(qr.QrError):
        qr.qr_rank(hq, q, np.zeros(10, np.uint8), o4[:10])      # mixed host/device pointers


def test_edge_cases_and_contract(cuda):
    """m = 0 is a no-op; q > n is memory-safe (clamped line); a cloned handle answers identically."""
    torch = _torch()
    n = 2 * S + 3
    w = gen.bits(5, n)
    h = qr.qr_birank_build(w, n)
    empty = torch.empty(0, dtype=torch.uint64, device=cuda)
    qr.qr_rank(h, empty, None, empty)                              # m = 0
    big = to_dev(np.array([n + 1, n + 496, 2 * n, (1 << 40)], np.uint64), cuda)
    ob = torch.empty_like(big)
    qr.qr_rank(h, big, None, ob)                                   # contract violation: must not fault
    qr.qr_sync()
    h2 = qr.qr_clone_to_device(h, 0)
    q = gen.queries(9, n, 50000)
    o1 = torch.empty(q.size, dtype=torch.uint64, device=cuda)
    o2 = torch.empty_like(o1)
    qr.qr_rank(h, to_dev(q, cuda), None, o1)
    qr.qr_rank(h2, to_dev(q, cuda), None, o2)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(o1), to_host(o2))
    assert np.array_equal(to_host(o1), oracle.BitsOracle(w, n).rank(q))
    n4 = 3 * S4 + 9
    t = gen.dna(6, n4)
    h4 = qr.qr_quadrank_build(t, n4)
    qb = to_dev(np.array([n4 + 1, 10 * n4], np.uint64), cuda)
    qr.qr_rank(h4, qb, to_dev(np.array([1, 3], np.uint8), cuda), torch.empty_like(qb))
    qr.qr_rank_all4(h4, qb, torch.empty((2, 4), dtype=torch.uint64, device=cuda))
    qr.qr_sync()
    fm = qr.qr_fm_build(t, n4)
    fm2 = qr.qr_fm_clone_to_device(fm, 0)
    pats = gen.patterns(2, 0, 3000, 20, t, n4)
    d1 = torch.empty(3000, dtype=torch.int32, device=cuda)
    d2 = torch.empty_like(d1)
    qr.qr_fm_count(fm, to_dev(pats, cuda), None, 20, d1, 3000)
    qr.qr_fm_count(fm2, to_dev(pats, cuda), None, 20, d2, 3000)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(d1), to_host(d2))
    assert fm2.C == fm.C and fm2.spos == fm.spos


@pytest.mark.parametrize("pair", [0, 1, 2])
def test_index64_path(cuda, pair):
    """The 64-bit line-index path (selected for n >= 2^36 / 2^37) forced on small n: bit-exact."""
    torch = _torch()
    n = 5 * S + 4321
    w, t = gen.bits(41, n), gen.dna(42, n)
    hb, hq = qr.qr_birank_build(w, n), qr.qr_quadrank_build(t, n)
    q, c = gen.queries(43, n, 100000, with_c=True)
    q = np.concatenate([q, boundary_queries(n, B, S, 240)])
    c = np.concatenate([c, (np.arange(q.size - c.size) % 4).astype(np.uint8)])
    dq, dc = to_dev(q, cuda), to_dev(c, cuda)
    ob, oq = torch.empty_like(dq), torch.empty_like(dq)
    o4 = torch.empty((q.size, 4), dtype=torch.uint64, device=cuda)
    qr.qr_set_tuning("index64", 1)
    qr.qr_set_tuning("rank_pair", pair)
    try:
        qr.qr_rank(hb, dq, None, ob)
        qr.qr_rank(hq, dq, dc, oq)
        qr.qr_rank_all4(hq, dq, o4)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("index64", 0)
        qr.qr_set_tuning("rank_pair", 2)
    assert np.array_equal(to_host(ob), oracle.BitsOracle(w, n).rank(q))
    ora = oracle.DnaOracle(t, n)
    assert np.array_equal(to_host(oq), ora.rank(q, c))
    assert np.array_equal(to_host(o4), ora.rank_all4(q))


def test_concurrent_streams_share_a_handle(cuda):
    """Handles are immutable: queries on several streams at once (and from the staged path on
    internal streams) give the same answers as one stream."""
    torch = _torch()
    n = 9 * S + 123
    w = gen.bits(51, n)
    h = qr.qr_birank_build(w, n)
    ref = None
    streams = [torch.cuda.Stream() for _ in range(4)]
    q = gen.queries(52, n, 400000)
    dq = to_dev(q, cuda)
    outs = [torch.empty_like(dq) for _ in streams]
    torch.cuda.synchronize()
    for s, o in zip(streams, outs):
        with torch.cuda.stream(s):
            qr.qr_rank(h, dq, None, o, stream=s)
    host_out = np.zeros(q.size, np.uint64)
    qr.qr_rank(h, q, None, host_out)
    torch.cuda.synchronize()
    qr.qr_sync()
    ref = oracle.BitsOracle(w, n).rank(q)
    for o in outs:
        assert np.array_equal(to_host(o), ref)
    assert np.array_equal(host_out, ref)


def test_concurrent_host_threads(cuda):
    """The header's promise: handles are usable from many host threads at once (ctypes drops the
    GIL inside the library).  Four threads, each on its own stream, run device-pointer rank
    batches (dynamic order: shared counter ring), staged host-pointer batches (shared internal
    streams) and FM counts against one BiRank and one FM handle; every result matches."""
    import threading

    import torch

    n = (1 << 27) + 5
    w = gen.bits(600, n)
    h = qr.qr_birank_build(w, n)
    ora = oracle.BitsOracle(w, n)
    nf = 100000
    tf = gen.dna(601, nf)
    fm = qr.qr_fm_build(tf, nf)
    L, mp = 20, 20000
    pats = gen.patterns(602, 0, mp, L, tf, nf)
    ref_fm = oracle.FmOracle(gen.unpack_dna(tf, nf)).count(pats, np.arange(mp, dtype=np.uint64) * L,
                                                          np.full(mp, L, np.uint32))
    errors = []

    def work(tid):
        try:
            s = torch.cuda.Stream()
            for it in range(3):
                m = (1 << 22) + 17 * tid + it
                q = gen.queries(610 + 10 * tid + it, n, m)
                dq = to_dev(q, cuda)
                out = torch.empty_like(dq)
                qr.qr_rank(h, dq, None, out, stream=s)
                hq = gen.queries(700 + 10 * tid + it, n, 300000)
                hout = np.zeros(hq.size, np.uint64)
                qr.qr_rank(h, hq, None, hout, stream=s)
                d = torch.empty(mp, dtype=torch.int32, device=cuda)
                qr.qr_fm_count(fm, to_dev(pats, cuda), None, L, d, mp, stream=s)
                s.synchronize()
                if not np.array_equal(to_host(out), ora.rank(q)):
                    errors.append((tid, it, "device rank"))
                if not np.array_equal(hout, ora.rank(hq)):
                    errors.append((tid, it, "staged rank"))
                if not np.array_equal(to_host(d).view(np.uint32), ref_fm):
                    errors.append((tid, it, "fm count"))
        except Exception as e:  # noqa: BLE001
            errors.append((tid, repr(e)))

    ts = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_gather_ceiling_rank4_shape(cuda):
    """qr_gather_ceiling mode 4 (QuadRank16): rank_4's loads and its 32-B output per query — lane 0
    of a pair stores the XOR pairs of sector 0, lane 1 those of sector 1 when the query reads it."""
    torch = _torch()
    n = 5 * S4 + 321
    t = gen.dna(17, n)
    h = qr.qr_quadrank_build(t, n)
    lines, _ = qr.qr_export_layout(h)
    u64 = lines.view(np.uint64).reshape(-1, 8)
    q = gen.queries(18, n, 60000)
    dq = to_dev(q, cuda)
    out = torch.zeros((q.size, 4), dtype=torch.uint64, device=cuda)
    qr.qr_gather_ceiling(h, dq, out, 4)
    torch.cuda.synchronize()
    j = (q // B4).astype(np.int64)
    right = (32 + q - j.astype(np.uint64) * B4) >= 128
    exp = np.stack([u64[j, 0] ^ u64[j, 1], u64[j, 2] ^ u64[j, 3],
                    np.where(right, u64[j, 4] ^ u64[j, 5], 0).astype(np.uint64),
                    np.where(right, u64[j, 6] ^ u64[j, 7], 0).astype(np.uint64)], axis=1)
    assert np.array_equal(to_host(out), exp)
    with pytest.raises(qr.QrError):                       # QuadRank16 only
        hb = qr.qr_birank_build(gen.bits(3, 5000), 5000)
        qr.qr_gather_ceiling(hb, dq[:10], torch.zeros((10, 4), dtype=torch.uint64, device=cuda), 4)


@pytest.mark.parametrize("space", ["device", "host"])
def test_opt_in_range_check(cuda, space):
    """check_range = 1 (reading R12: rank is defined for 0 <= q <= n): qr_rank and
    qr_rank_all4 count the queries with q > n, still answer the valid ones exactly, and return
    QR_ERANGE naming the count; q = n is in range; off (default) the same call returns QR_OK."""
    torch = _torch()
    n = 3 * S + 17
    w = gen.bits(7, n)
    h = qr.qr_birank_build(w, n)
    n4 = 2 * S4 + 5
    t = gen.dna(8, n4)
    h4 = qr.qr_quadrank_build(t, n4)
    q = gen.queries(10, n, 100000)
    q[[5, 77, 99999]] = [n + 1, 2 * n, 1 << 50]
    q[6] = n
    bad = np.flatnonzero(q > n)
    good = np.setdiff1d(np.arange(q.size), bad)
    q4 = gen.queries(11, n4, 50000)
    q4[[0, 1]] = [n4 + 1, n4 + 224]
    c4 = np.zeros(q4.size, np.uint8)
    dev = space == "device"
    qq, q44 = (to_dev(q, cuda), to_dev(q4, cuda)) if dev else (q, q4)
    out = torch.empty(q.size, dtype=torch.uint64, device=cuda) if dev else np.zeros(q.size, np.uint64)
    o4 = torch.empty((q4.size, 4), dtype=torch.uint64, device=cuda) if dev else np.zeros((q4.size, 4), np.uint64)
    cc = to_dev(c4, cuda) if dev else c4
    o1 = torch.empty(q4.size, dtype=torch.uint64, device=cuda) if dev else np.zeros(q4.size, np.uint64)
    qr.qr_set_tuning("check_range", 1)
    try:
        with pytest.raises(qr.QrError) as e:
            qr.qr_rank(h, qq, None, out)
        assert e.value.status == qr.QR_ERANGE and "3 of the queries" in str(e.value)
        with pytest.raises(qr.QrError) as e:
            qr.qr_rank_all4(h4, q44, o4)
        assert e.value.status == qr.QR_ERANGE and "2 of the queries" in str(e.value)
        with pytest.raises(qr.QrError) as e:
            qr.qr_rank(h4, q44, cc, o1)
        assert e.value.status == qr.QR_ERANGE
        qok = q[good].copy()
        ook = np.zeros(qok.size, np.uint64)
        qr.qr_rank(h, qok, None, ook)                          # all in range (incl. q = n): QR_OK
    finally:
        qr.qr_set_tuning("check_range", 0)
    torch.cuda.synchronize()
    res = to_host(out) if dev else out
    assert np.array_equal(res[good], oracle.BitsOracle(w, n).rank(q[good]))
    assert np.array_equal(ook, oracle.BitsOracle(w, n).rank(qok))
    r4 = to_host(o4) if dev else o4
    assert np.array_equal(r4[2:], oracle.DnaOracle(t, n4).rank_all4(q4[2:]))
    qr.qr_rank(h, qq, None, out)                               # default: no check, QR_OK
    qr.qr_sync()
