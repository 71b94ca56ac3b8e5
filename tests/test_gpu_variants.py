"""GPU parity of the no-L1-array layout variants (NEXT §8(f)4): BiRank64x2 and
QuadRank64 against the same oracle, bit-exact, incl. the sector / line
boundaries (192, 384 bits; 64, 128 chars), ragged tails and the host-pointer path."""
import numpy as np
import pytest

import gen
import oracle
import paper_2602_04103_b200 as qr
from _util import boundary_queries, to_dev, to_host

pytestmark = pytest.mark.gpu

B64_SIZES = [0, 1, 95, 96, 97, 191, 192, 193, 383, 384, 385, 5000, 3 * 384 * 1000 + 77, (1 << 22) + 3]
Q64_SIZES = [0, 1, 63, 64, 65, 127, 128, 129, 3000, 128 * 5000 + 31, (1 << 21) + 5]


def _torch():
    import torch

    return torch


@pytest.mark.parametrize("n", B64_SIZES)
@pytest.mark.parametrize("p", [0.5, 1.0])
def test_birank64x2_parity(cuda, n, p):
    torch = _torch()
    w = gen.bits(3000 + n, n, p)
    h = qr.qr_build(w, n, qr.QR_LAYOUT_BIRANK64X2)
    assert h.layout == qr.QR_LAYOUT_BIRANK64X2 and h.super_bytes == 0
    assert h.line_bytes == 64 * (n // 384 + 1)
    ora = oracle.BitsOracle(w, n)
    q = np.arange(n + 1, dtype=np.uint64) if n <= 100000 else \
        np.concatenate([gen.queries(1, n, 200000), boundary_queries(n, 192, 384, 96)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, out)
    c = (gen.queries(2, 1, q.size, with_c=True)[1] & 1).astype(np.uint8)
    out2 = torch.empty_like(dq)
    qr.qr_rank(h, dq, to_dev(c, cuda), out2)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), ora.rank(q))
    assert np.array_equal(to_host(out2), ora.rank(q, c))


@pytest.mark.parametrize("n", Q64_SIZES)
def test_quadrank64_parity(cuda, n):
    torch = _torch()
    w = gen.dna(4000 + n, n)
    h = qr.qr_build(w, n, qr.QR_LAYOUT_QUADRANK64)
    assert h.layout == qr.QR_LAYOUT_QUADRANK64 and h.super_bytes == 0
    ora = oracle.DnaOracle(w, n)
    if n <= 40000:
        q = np.repeat(np.arange(n + 1, dtype=np.uint64), 4)
        c = np.tile(np.arange(4, dtype=np.uint8), n + 1)
    else:
        q, c = gen.queries(5, n, 200000, with_c=True)
        q = np.concatenate([q, boundary_queries(n, 64, 128, 0)])
        c = np.concatenate([c, (np.arange(q.size - c.size) % 4).astype(np.uint8)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, to_dev(c, cuda), out)
    qu = np.unique(q)
    o4 = torch.empty((qu.size, 4), dtype=torch.uint64, device=cuda)
    qr.qr_rank_all4(h, to_dev(qu, cuda), o4)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), ora.rank(q, c))
    assert np.array_equal(to_host(o4), ora.rank_all4(qu))


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_variants_tuning_and_host_path(cuda, k):
    torch = _torch()
    n = 777777
    wb, wd = gen.bits(8, n), gen.dna(9, n)
    hb = qr.qr_build(to_dev(wb, cuda), n, qr.QR_LAYOUT_BIRANK64X2)
    hq = qr.qr_build(to_dev(wd, cuda), n, qr.QR_LAYOUT_QUADRANK64)
    q, c = gen.queries(10, n, 123457, with_c=True)
    qr.qr_set_tuning("rank_k", k)
    try:
        ob, oq = np.zeros(q.size, np.uint64), np.zeros(q.size, np.uint64)
        o4 = np.zeros((q.size, 4), np.uint64)
        qr.qr_rank(hb, q, None, ob)
        qr.qr_rank(hq, q, c, oq)
        qr.qr_rank_all4(hq, q, o4)
        qr.qr_sync()
        big = to_dev(np.array([n + 1, 5 * n, 1 << 40], np.uint64), cuda)      # q > n: memory-safe
        qr.qr_rank(hb, big, None, torch.empty_like(big))
        qr.qr_rank(hq, big, to_dev(np.zeros(3, np.uint8), cuda), torch.empty_like(big))
        g = torch.empty(q.size, dtype=torch.uint64, device=cuda)
        qr.qr_gather_ceiling(hq, to_dev(q, cuda), g, 0)
        qr.qr_sync()
    finally:
        qr.qr_set_tuning("rank_k", 2)
    assert np.array_equal(ob, oracle.BitsOracle(wb, n).rank(q))
    oraq = oracle.DnaOracle(wd, n)
    assert np.array_equal(oq, oraq.rank(q, c))
    assert np.array_equal(o4, oraq.rank_all4(q))
    lines, _ = qr.qr_export_layout(hq)
    u64 = lines.view(np.uint64).reshape(-1, 8)
    assert np.array_equal(to_host(g), np.bitwise_xor.reduce(u64[(q >> np.uint64(7)).astype(np.int64)], axis=1))
    with pytest.raises(qr.QrError):
        qr.qr_build(wb, n, 99)


def _chain_reference(rank_fn, q, n, L):
    """Host simulation of the dependent chains with the oracle (SPEC S:413 rule)."""
    m = q.size
    out = np.zeros(m, np.uint64)
    chains = (m + L - 1) // L
    qq = np.zeros((chains, L), np.uint64)
    valid = np.zeros((chains, L), bool)
    flat = np.arange(chains * L)
    qq.reshape(-1)[: m] = q
    valid.reshape(-1)[: m] = True
    r = np.zeros(chains, np.uint64)
    for i in range(L):
        qe = qq[:, i] + r
        qe = np.where(qe >= n + 1, qe - np.uint64(n + 1), qe)
        ri = rank_fn(qe, i)
        r = np.where(valid[:, i], ri, r)
        idx = np.arange(chains) * L + i
        ok = idx < m
        out[idx[ok]] = ri[ok]
    del flat
    return out


@pytest.mark.parametrize("layout", [qr.QR_LAYOUT_BIRANK16, qr.QR_LAYOUT_BIRANK64X2, qr.QR_LAYOUT_QUADRANK16,
                                    qr.QR_LAYOUT_QUADRANK64, qr.QR_LAYOUT_BIRANK16X2, qr.QR_LAYOUT_QUADRANK16X2,
                                    qr.QR_LAYOUT_BIRANK32X2])
def test_rank_chain_latency_mode(cuda, layout):
    torch = _torch()
    n = 3 * 63488 + 1001
    bits = layout in (qr.QR_LAYOUT_BIRANK16, qr.QR_LAYOUT_BIRANK64X2, qr.QR_LAYOUT_BIRANK16X2, qr.QR_LAYOUT_BIRANK32X2)
    w = gen.bits(21, n) if bits else gen.dna(22, n)
    h = qr.qr_build(w, n, layout)
    m, L = 40003, 37                                  # ragged last chain
    q, c = gen.queries(23, n, m, with_c=True)
    if bits:
        ora = oracle.BitsOracle(w, n)
        ref = _chain_reference(lambda qe, i: ora.rank(qe), q, n, L)
        cdev = None
    else:
        ora = oracle.DnaOracle(w, n)
        cc = np.zeros(((m + L - 1) // L) * L, np.uint8)
        cc[:m] = c
        cm = cc.reshape(-1, L)
        ref = _chain_reference(lambda qe, i: ora.rank(qe, cm[:, i]), q, n, L)
        cdev = to_dev(c, cuda)
    out = torch.empty(m, dtype=torch.uint64, device=cuda)
    qr.qr_rank_chain(h, to_dev(q, cuda), cdev, out, L)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), ref)


@pytest.mark.parametrize("layout", [qr.QR_LAYOUT_BIRANK16, qr.QR_LAYOUT_BIRANK64X2, qr.QR_LAYOUT_QUADRANK16,
                                    qr.QR_LAYOUT_QUADRANK64, qr.QR_LAYOUT_BIRANK16X2, qr.QR_LAYOUT_QUADRANK16X2,
                                    qr.QR_LAYOUT_BIRANK32X2])
def test_save_load_roundtrip(cuda, layout, tmp_path):
    """Checkpoint/resume: export -> .npz -> import gives a handle that answers identically, and the
    build is deterministic (byte-identical layout on a rebuild)."""
    torch = _torch()
    n = 2 * 63488 * 2 + 999
    bits = layout in (qr.QR_LAYOUT_BIRANK16, qr.QR_LAYOUT_BIRANK64X2, qr.QR_LAYOUT_BIRANK16X2, qr.QR_LAYOUT_BIRANK32X2)
    w = gen.bits(31, n) if bits else gen.dna(32, n)
    h = qr.qr_build(w, n, layout)
    p = str(tmp_path / "idx.npz")
    qr.save_index(h, p)
    h2 = qr.load_index(p)
    assert (h2.n, h2.layout, h2.line_bytes, h2.super_bytes) == (h.n, h.layout, h.line_bytes, h.super_bytes)
    l1, s1 = qr.qr_export_layout(h)
    l3, s3 = qr.qr_export_layout(qr.qr_build(w, n, layout))
    assert np.array_equal(l1, l3) and np.array_equal(s1, s3)
    q, c = gen.queries(33, n, 50000, with_c=True)
    dq = to_dev(q, cuda)
    dc = None if bits else to_dev(c, cuda)
    o1, o2 = torch.empty_like(dq), torch.empty_like(dq)
    qr.qr_rank(h, dq, dc, o1)
    qr.qr_rank(h2, dq, dc, o2)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(o1), to_host(o2))


# ------------------------------------------------------------------ BiRank16x2
B16X2_SIZES = [0, 1, 119, 120, 121, 239, 240, 241, 359, 360, 361, 479, 480, 481, 959, 960, 961,
               128 * 480 - 1, 128 * 480, 128 * 480 + 1, 6 * 128 * 480 + 7, 13 * 128 * 480 + 3333, (1 << 22) + 3]


@pytest.mark.parametrize("n", B16X2_SIZES)
@pytest.mark.parametrize("p", [0.5, 1.0, 0.01])
def test_birank16x2_parity(cuda, n, p):
    """BiRank16x2: every q on small n, boundaries of the 1/4 / 3/4 anchors (120, 360), the sector
    split (240), lines (480) and superblocks (128 lines) on larger n; all-ones makes every delta
    and superblock increment maximal; rank with c (c = 0 -> q - rank)."""
    torch = _torch()
    w = gen.bits(5000 + n, n, p)
    h = qr.qr_build(w, n, qr.QR_LAYOUT_BIRANK16X2)
    L = n // 480 + 1
    assert h.layout == qr.QR_LAYOUT_BIRANK16X2
    assert h.line_bytes == 64 * L and h.super_bytes == 4 * ((L - 1) // 128 + 1)
    ora = oracle.BitsOracle(w, n)
    if n <= 100000:
        q = np.arange(n + 1, dtype=np.uint64)
    else:
        q = np.concatenate([gen.queries(6, n, 200000), boundary_queries(n, 240, 128 * 480, 120)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, out)
    c = (gen.queries(7, 1, q.size, with_c=True)[1] & 1).astype(np.uint8)
    out2 = torch.empty_like(dq)
    qr.qr_rank(h, dq, to_dev(c, cuda), out2)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), ora.rank(q))
    assert np.array_equal(to_host(out2), ora.rank(q, c))


def test_birank16x2_layout_closed_forms(cuda):
    """Decode every sector: d_{j,h} + 2^11 s_{j>>7} = rank(480 j + 240 h + 120) (the 1/4 and 3/4
    anchors), s_i = rank(128 i * 480) >> 11, data = text u16 words; byte
    accounting 6.72% at n = 2^34."""
    for n, p in [(9 * 128 * 480 + 1234, 0.5), (3 * 128 * 480 + 17, 1.0)]:
        w = gen.bits(77, n, p)
        h = qr.qr_build(w, n, qr.QR_LAYOUT_BIRANK16X2)
        lines, sup = qr.qr_export_layout(h)
        L = n // 480 + 1
        u16 = lines.view(np.uint16).reshape(L, 2, 16)
        ora = oracle.BitsOracle(w, n)
        for hh in (0, 1):
            anchors = np.minimum(np.arange(L, dtype=np.uint64) * 480 + 240 * hh + 120, n)
            d = u16[:, hh, 0].astype(np.uint64) + (sup[np.arange(L) // 128].astype(np.uint64) << 11)
            assert np.array_equal(d, ora.rank(anchors)), hh
        sb = np.minimum(np.arange(sup.size, dtype=np.uint64) * 128 * 480, n)
        assert np.array_equal(sup.astype(np.uint64), ora.rank(sb) >> 11)
        text16 = np.zeros(30 * L, np.uint16)
        t = w.view(np.uint16)[: min(w.size * 4, 30 * L)]
        text16[: t.size] = t
        assert np.array_equal(u16[:, :, 1:].reshape(-1), text16)
    n = 1 << 34
    L = n // 480 + 1
    overhead = (64 * L + 4 * ((L - 1) // 128 + 1)) * 8 / n - 1
    assert abs(overhead - 0.0672) < 0.0005


@pytest.mark.parametrize("src", ["table", "global", "cluster"])
def test_birank16x2_superblock_sources(cuda, src):
    """The three superblock-word sources (per-CTA table, L2, 2-CTA cluster shared memory) and the
    dynamic order on a batch >= 2^22; the gather ceiling loads the query's sector."""
    torch = _torch()
    knobs = {"table": [("rank_lane_table", 1), ("rank_smem", 0)], "global": [("rank_lane_table", 0), ("rank_smem", 0)],
             "cluster": [("rank_smem", 2)]}[src]
    n = 23 * 128 * 480 + 999
    w = gen.bits(88, n)
    h = qr.qr_build(w, n, qr.QR_LAYOUT_BIRANK16X2)
    m = (1 << 22) + 17
    q = gen.queries(89, n, m)
    dq = to_dev(q, cuda)
    try:
        for k, v in knobs:
            qr.qr_set_tuning(k, v)
        out = torch.empty_like(dq)
        qr.qr_rank(h, dq, None, out)
        c = (gen.queries(90, 1, m, with_c=True)[1] & 1).astype(np.uint8)
        out2 = torch.empty_like(dq)
        qr.qr_rank(h, dq, to_dev(c, cuda), out2)
        g = torch.empty_like(dq)
        qr.qr_gather_ceiling(h, dq, g, 0)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("rank_lane_table", 1)
        qr.qr_set_tuning("rank_smem", 1)
    ora = oracle.BitsOracle(w, n)
    assert np.array_equal(to_host(out), ora.rank(q))
    assert np.array_equal(to_host(out2), ora.rank(q, c))


# ------------------------------------------------------------------ QuadRank16x2 (B200 sector-local σ=4 variant)
Q16X2_SIZES = [0, 1, 47, 48, 49, 95, 96, 97, 143, 144, 145, 191, 192, 193, 383, 384, 385,
               256 * 192 - 1, 256 * 192, 256 * 192 + 1, 9 * 256 * 192 + 77, 17 * 256 * 192 + 4321, (1 << 21) + 5]


def _q16x2_text(kind, n, seed):
    if kind == "iid":
        return gen.dna(seed, n)
    word = {"G": 0xAAAAAAAAAAAAAAAA, "T": 0xFFFFFFFFFFFFFFFF}[kind]
    return np.full(max(1, (n + 31) // 32), np.uint64(word))


@pytest.mark.parametrize("n", Q16X2_SIZES)
@pytest.mark.parametrize("kind", ["iid", "G"])
def test_quadrank16x2_parity(cuda, n, kind):
    """rank(q,c) for every (q,c) on small n, boundaries of the sector anchors (48, 144), the sector
    split (96), lines (192) and superblocks (256 lines) on larger n; rank_4; a single repeated
    symbol makes every delta and superblock increment maximal."""
    torch = _torch()
    w = _q16x2_text(kind, n, 6000 + n)
    h = qr.qr_build(w, n, qr.QR_LAYOUT_QUADRANK16X2)
    L = n // 192 + 1
    assert h.layout == qr.QR_LAYOUT_QUADRANK16X2
    assert h.line_bytes == 64 * L and h.super_bytes == 16 * ((L - 1) // 256 + 1)
    ora = oracle.DnaOracle(w, n)
    if n <= 40000:
        q = np.repeat(np.arange(n + 1, dtype=np.uint64), 4)
        c = np.tile(np.arange(4, dtype=np.uint8), n + 1)
    else:
        q, c = gen.queries(8, n, 200000, with_c=True)
        bq = boundary_queries(n, 96, 256 * 192, 48)
        q = np.concatenate([q, np.repeat(bq, 4)])
        c = np.concatenate([c, np.tile(np.arange(4, dtype=np.uint8), bq.size)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, to_dev(c, cuda), out)
    o4 = torch.empty((q.size, 4), dtype=torch.uint64, device=cuda)
    qr.qr_rank_all4(h, dq, o4)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), ora.rank(q, c))
    assert np.array_equal(to_host(o4), ora.rank_all4(q))


def test_quadrank16x2_layout_closed_forms(cuda):
    """Decode every sector: d_{j,h,c} + 2^13 s_{j>>8,c} = rank(192 j + 96 h + 48, c), s_{i,c} =
    rank(256 i 192, c) >> 13, data = the bit planes of text chars 192 j + 96 h .. +96 (low / high
    planes of chars 0..63 in words 1 / 2, both planes of chars 64..95 in word 3)."""
    for n in (11 * 256 * 192 + 999, 2 * 256 * 192 + 5):
        w = gen.dna(91, n)
        h = qr.qr_build(w, n, qr.QR_LAYOUT_QUADRANK16X2)
        lines, sup = qr.qr_export_layout(h)
        L = n // 192 + 1
        u64 = lines.view(np.uint64).reshape(L, 2, 4)
        sup = sup.view(np.uint32).reshape(-1, 4)
        ora = oracle.DnaOracle(w, n)
        for hh in (0, 1):
            raw = np.arange(L, dtype=np.uint64) * 192 + 96 * hh + 48
            anchors = np.minimum(raw, n)
            for c in range(4):
                d = (u64[:, hh, 0] >> np.uint64(16 * c)) & np.uint64(0xffff)
                full = d + (sup[np.arange(L) // 256, c].astype(np.uint64) << np.uint64(13))
                # an anchor past n counts the padding characters, which are A (reading R4)
                want = ora.rank(anchors, np.full(L, c, np.uint8)) + (raw - anchors if c == 0 else 0)
                assert np.array_equal(full, want), (hh, c)
        text = np.zeros(6 * L, np.uint64)
        text[: min(w.size, 6 * L)] = w[: 6 * L]
        chars = gen.unpack_dna(text, 192 * L).reshape(L, 2, 96).astype(np.uint64)
        bitpos = np.uint64(1) << np.arange(64, dtype=np.uint64)
        lo = ((chars & 1)[..., :64] * bitpos).sum(axis=-1, dtype=np.uint64)
        hi = ((chars >> 1)[..., :64] * bitpos).sum(axis=-1, dtype=np.uint64)
        p2 = ((chars & 1)[..., 64:] * bitpos[:32]).sum(axis=-1, dtype=np.uint64) | \
            (((chars >> 1)[..., 64:] * bitpos[:32]).sum(axis=-1, dtype=np.uint64) << np.uint64(32))
        assert np.array_equal(u64[:, :, 1], lo) and np.array_equal(u64[:, :, 2], hi) and np.array_equal(u64[:, :, 3], p2)


@pytest.mark.parametrize("src", ["table", "global", "cluster"])
def test_quadrank16x2_superblock_sources(cuda, src):
    torch = _torch()
    knobs = {"table": [("rank_lane_table", 1), ("rank_smem", 0)], "global": [("rank_lane_table", 0), ("rank_smem", 0)],
             "cluster": [("rank_smem", 2)]}[src]
    n = 21 * 256 * 192 + 321
    w = gen.dna(92, n)
    h = qr.qr_build(w, n, qr.QR_LAYOUT_QUADRANK16X2)
    m = (1 << 22) + 9
    q, c = gen.queries(93, n, m, with_c=True)
    dq = to_dev(q, cuda)
    try:
        for k, v in knobs:
            qr.qr_set_tuning(k, v)
        out = torch.empty_like(dq)
        qr.qr_rank(h, dq, to_dev(c, cuda), out)
        o4 = torch.empty((m, 4), dtype=torch.uint64, device=cuda)
        qr.qr_rank_all4(h, dq, o4)
        g = torch.empty_like(dq)
        qr.qr_gather_ceiling(h, dq, g, 0)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("rank_lane_table", 1)
        qr.qr_set_tuning("rank_smem", 1)
    ora = oracle.DnaOracle(w, n)
    assert np.array_equal(to_host(out), ora.rank(q, c))
    assert np.array_equal(to_host(o4), ora.rank_all4(q))


# ------------------------------------------------------------------ BiRank32x2
B32X2_SIZES = [0, 1, 111, 112, 113, 223, 224, 225, 335, 336, 337, 447, 448, 449, 895, 896, 897,
               5000, 3 * 448 * 1000 + 77, (1 << 22) + 3]


@pytest.mark.parametrize("n", B32X2_SIZES)
@pytest.mark.parametrize("p", [0.5, 1.0, 0.01])
def test_birank32x2_parity(cuda, n, p):
    """BiRank32x2: every q on small n, the anchors (112, 336), the sector split (224) and lines
    (448) on larger n; rank with c."""
    torch = _torch()
    w = gen.bits(7000 + n, n, p)
    h = qr.qr_build(w, n, qr.QR_LAYOUT_BIRANK32X2)
    L = n // 448 + 1
    assert h.layout == qr.QR_LAYOUT_BIRANK32X2
    assert h.line_bytes == 64 * L and h.super_bytes == 8 * ((L - 1) // (1 << 23) + 1)
    ora = oracle.BitsOracle(w, n)
    q = np.arange(n + 1, dtype=np.uint64) if n <= 100000 else \
        np.concatenate([gen.queries(9, n, 200000), boundary_queries(n, 224, 448 * 1000, 112)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, out)
    c = (gen.queries(10, 1, q.size, with_c=True)[1] & 1).astype(np.uint8)
    out2 = torch.empty_like(dq)
    qr.qr_rank(h, dq, to_dev(c, cuda), out2)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), ora.rank(q))
    assert np.array_equal(to_host(out2), ora.rank(q, c))


def test_birank32x2_layout_and_l1_boundary(cuda):
    """Decode sectors (d_{j,h} + L1[j >> 23] = rank(448 j + 224 h + 112)); a 2^32 + 5-bit text
    crosses the first L1 boundary (2^23 lines = 3.76e9 bits): queries around it and uniform ones,
    dynamic order (m >= 2^22), vs the oracle."""
    torch = _torch()
    n = 9 * 448 + 100
    w = gen.bits(3, n, 0.5)
    h = qr.qr_build(w, n, qr.QR_LAYOUT_BIRANK32X2)
    lines, l1 = qr.qr_export_layout(h)
    L = n // 448 + 1
    u32 = lines.view(np.uint32).reshape(L, 2, 8)
    ora = oracle.BitsOracle(w, n)
    for hh in (0, 1):
        anchors = np.minimum(np.arange(L, dtype=np.uint64) * 448 + 224 * hh + 112, n)
        assert np.array_equal(u32[:, hh, 0].astype(np.uint64) + l1.view(np.uint64)[0], ora.rank(anchors))
    n = (1 << 32) + 5
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=cuda)
    gen.bits_dev(11, n, 0.5, bits)
    h = qr.qr_build(bits, n, qr.QR_LAYOUT_BIRANK32X2)
    assert h.super_bytes == 16
    wh = bits.cpu().numpy()
    del bits
    ora = oracle.BitsOracle(wh, n)
    edge = 448 * (1 << 23)
    qe = np.arange(edge - 2000, edge + 2000, dtype=np.uint64)
    m = (1 << 22) + 11
    q = np.concatenate([gen.queries(12, n, m - qe.size - 2), qe, np.array([0, n], np.uint64)])
    dq = to_dev(q, cuda)
    out = torch.empty_like(dq)
    qr.qr_rank(h, dq, None, out)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), ora.rank(q))
