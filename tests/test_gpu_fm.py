"""GPU parity of QuadFm (App. D) against the CPU oracle: GPU-built suffix array /
BWT / C / spos, the BWT QuadRank, the 8-mer table, and fm_count on exact, random, short,
empty, seeded-length and longer-than-text patterns.  Bit-exact (u32 counts)."""
import itertools

import numpy as np
import pytest

import gen
import oracle
import paper_2602_04103_b200 as qr
from _util import to_dev, to_host

pytestmark = pytest.mark.gpu
DEFAULT_FM_STEP = 0


def _torch():
    import torch

    return torch


@pytest.fixture
def fm_dyn_reset():
    yield
    qr.qr_set_tuning("fm_dyn", 1)
    qr.qr_set_tuning("fm_step", DEFAULT_FM_STEP)


def pack2(sym: np.ndarray) -> np.ndarray:
    n = sym.size
    w = np.zeros((n + 31) // 32 + 1, np.uint64)
    s = np.zeros(((n + 31) // 32) * 32, np.uint64)
    s[:n] = sym
    s = s.reshape(-1, 32)
    w[: s.shape[0]] = (s << (2 * np.arange(32, dtype=np.uint64))).sum(axis=1, dtype=np.uint64)
    return w


def mixed_patterns(rng, sym, count):
    n = sym.size
    pats = []
    for i in range(count):
        kind = i % 5
        if kind == 0:                                   # exact substring, any length
            L = int(rng.integers(1, 60)); a = int(rng.integers(0, max(1, n - L + 1)))
            pats.append(sym[a:a + L].copy())
        elif kind == 1:                                 # random, short (< 8: no seeding)
            pats.append(rng.integers(0, 4, int(rng.integers(0, 8))).astype(np.uint8))
        elif kind == 2:                                 # exactly 8 (seed only), 9
            pats.append(rng.integers(0, 4, 8 + int(rng.integers(0, 2))).astype(np.uint8))
        elif kind == 3:                                 # random long
            pats.append(rng.integers(0, 4, int(rng.integers(8, 40))).astype(np.uint8))
        else:                                           # exact with one substitution
            L = int(rng.integers(10, 50)); a = int(rng.integers(0, max(1, n - L + 1)))
            p = sym[a:a + L].copy()
            if p.size:
                k = int(rng.integers(0, p.size)); p[k] = (p[k] + 1 + rng.integers(0, 3)) % 4
            pats.append(p)
    pats.append(sym.copy())                             # whole text
    pats.append(np.concatenate([sym, sym[:3]]))          # longer than the text
    pats.append(np.zeros(0, np.uint8))                   # empty -> n+1
    return pats


@pytest.mark.parametrize("n,kind", [(1, 0), (2, 0), (7, 0), (31, 0), (100, 0), (224, 0), (1000, 0), (50000, 0),
                                    (131072 + 123, 0), (25000, 1), (200000, 1)])
def test_fm_build_and_count_parity(cuda, n, kind):
    torch = _torch()
    w = gen.dna(300 + n, n, kind)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    fm = qr.qr_fm_build(w, n)
    # SA-derived quantities (GPU prefix doubling vs oracle doubling + qsort)
    assert fm.spos == ora.spos
    assert fm.C == [int(x) for x in ora.C]
    # the BWT rank structure ('$' stored as A) vs the oracle BWT with '$' -> A
    bw = ora.bwt.copy(); bw[bw == 4] = 0
    bora = oracle.DnaOracle(pack2(bw), n + 1)
    if n < 20000:                                               # every q in [0, N], every c
        q = np.repeat(np.arange(n + 2, dtype=np.uint64), 4)
        c = np.tile(np.arange(4, dtype=np.uint8), n + 2)
    else:
        q, c = gen.queries(1, n + 1, 100000, with_c=True)
    out = torch.empty(q.size, dtype=torch.uint64, device=cuda)
    qr.qr_rank(fm.bwt, to_dev(q, cuda), to_dev(c, cuda), out)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), bora.rank(q, c))
    # counts
    rng = np.random.default_rng(n)
    pats = mixed_patterns(rng, sym, 600)
    cat, off, lens = oracle.pack_patterns(pats)
    ref = ora.count(cat, off, lens)
    if n <= 1000:
        brute = np.array([sum(1 for i in range(n - len(p) + 1) if np.array_equal(sym[i:i + len(p)], p)) if len(p) else n + 1
                          for p in pats], np.uint32)
        assert np.array_equal(ref, brute)
    dout = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, dout, lens.size)
    torch.cuda.synchronize()
    got = to_host(dout).view(np.uint32)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"n={n}: {bad.size} mismatches: idx={bad[:5]} got={got[bad[:5]]} ref={ref[bad[:5]]}"
    # host-pointer path with variable lengths
    hout = np.zeros(lens.size, np.uint32)
    qr.qr_fm_count(fm, cat, lens, 0, hout, lens.size)
    qr.qr_sync()
    assert np.array_equal(hout, ref)


def _repetitive(name: str, n: int) -> np.ndarray:
    rng = np.random.default_rng(n)
    if name == "all_A":
        return np.zeros(n, np.uint8)
    if name == "all_T":
        return np.full(n, 3, np.uint8)
    if name == "period4":
        return np.resize(np.array([0, 1, 2, 3], np.uint8), n)
    if name == "period2_tail":                     # (AC)^k then one G: every group splits late
        s = np.resize(np.array([0, 1], np.uint8), n); s[-1] = 2
        return s
    if name == "period37":
        return np.resize(rng.integers(0, 4, 37).astype(np.uint8), n)
    if name == "doubled":                          # a random half repeated: groups of two to the end
        h = rng.integers(0, 4, n // 2).astype(np.uint8)
        return np.concatenate([h, h, rng.integers(0, 4, n - 2 * (n // 2)).astype(np.uint8)])
    raise ValueError(name)


@pytest.mark.parametrize("name", ["all_A", "all_T", "period4", "period2_tail", "period37", "doubled"])
@pytest.mark.parametrize("n", [1, 21, 22, 43, 1000, 6001])
def test_fm_build_repetitive_texts(cuda, name, n):
    """The GPU suffix sort (prefix doubling with discarding) on texts whose suffix groups stay
    large for many rounds: the BWT, spos and C must equal the oracle's (which sorts by doubling +
    qsort), checked through the BWT rank at every q and c, plus counts of every pattern shape."""
    torch = _torch()
    sym = _repetitive(name, n)
    w = pack2(sym)
    ora = oracle.FmOracle(sym)
    fm = qr.qr_fm_build(w, n)
    assert fm.spos == ora.spos
    assert fm.C == [int(x) for x in ora.C]
    bw = ora.bwt.copy(); bw[bw == 4] = 0
    bora = oracle.DnaOracle(pack2(bw), n + 1)
    q = np.repeat(np.arange(n + 2, dtype=np.uint64), 4)
    c = np.tile(np.arange(4, dtype=np.uint8), n + 2)
    out = torch.empty(q.size, dtype=torch.uint64, device=cuda)
    qr.qr_rank(fm.bwt, to_dev(q, cuda), to_dev(c, cuda), out)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(out), bora.rank(q, c))
    pats = mixed_patterns(np.random.default_rng(7), sym, 200)
    cat, off, lens = oracle.pack_patterns(pats)
    ref = ora.count(cat, off, lens)
    dout = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, dout, lens.size)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(dout).view(np.uint32), ref)


def test_fm_kmer_table_matches_oracle(cuda):
    n = 300000
    w = gen.dna(42, n)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    fm = qr.qr_fm_build(w, n, kmer_k=8)
    t = qr.qr_fm_export_kmer(fm)
    # key: 2 bits per char, last pattern char in the low bits
    keys = np.arange(65536, dtype=np.uint32)
    pats = np.stack([(keys >> (2 * (7 - i))) & 3 for i in range(8)], axis=1).astype(np.uint8)
    cat = np.ascontiguousarray(pats.reshape(-1))
    off = np.arange(65536, dtype=np.uint64) * 8
    lens = np.full(65536, 8, np.uint32)
    ref = ora.count(cat, off, lens)
    size = (t[:, 1].astype(np.int64) - t[:, 0].astype(np.int64))
    assert np.array_equal(size, ref.astype(np.int64))
    assert int(ref.sum()) == n - 7                               # partition identity
    # lo of a non-empty interval = C[c_last] + ... : check monotone order of the 4^8 intervals
    nz = size > 0
    order = np.argsort(t[nz, 0])
    assert np.all(np.diff(t[nz, 0][order].astype(np.int64)) > 0)


def test_fm_given_sa_and_fixed_length_and_work(cuda):
    torch = _torch()
    n = 120000
    w = gen.dna(77, n)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    fm_gpu_sa = qr.qr_fm_build(w, n)
    fm_given = qr.qr_fm_build(to_dev(w, cuda), n, sa=ora.sa)      # caller-provided SA (host)
    L, m = 32, 20000
    pats = gen.patterns(5, 0, m, L, w, n)
    off = np.arange(m, dtype=np.uint64) * L
    lens = np.full(m, L, np.uint32)
    ref = ora.count(pats, off, lens)
    assert np.all(ref[0::2] >= 1)                               # exact substrings occur
    for fm in (fm_gpu_sa, fm_given):
        d = torch.empty(m, dtype=torch.int32, device=cuda)
        qr.qr_fm_count(fm, to_dev(pats, cuda), None, L, d, m)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(d).view(np.uint32), ref)
    work = torch.zeros(2, dtype=torch.uint64, device=cuda)
    d = torch.empty(m, dtype=torch.int32, device=cuda)
    qr.qr_fm_count_work(fm_gpu_sa, to_dev(pats, cuda), None, L, d, m, work)
    torch.cuda.synchronize()
    ts, tl = ora.work(pats, off, lens, skip=8, block=224)
    assert [int(x) for x in to_host(work)] == [ts, tl]
    # host staged fixed-length path
    h = np.zeros(m, np.uint32)
    qr.qr_set_tuning("stage_chunk", 4096)
    try:
        qr.qr_fm_count(fm_gpu_sa, pats, None, L, h, m)
        qr.qr_sync()
    finally:
        qr.qr_set_tuning("stage_chunk", 1 << 23)
    assert np.array_equal(h, ref)


def test_fm_all_kmers_partition(cuda):
    torch = _torch()
    n = 40000
    w = gen.dna(8, n, 1 if n >= 2 * gen.BLOCK else 0)
    fm = qr.qr_fm_build(w, n)
    for k in (1, 2, 3, 9):
        pats = np.array(list(itertools.product(range(4), repeat=k)) if k < 9 else
                        np.random.default_rng(1).integers(0, 4, (5000, 9)), np.uint8)
        d = torch.empty(pats.shape[0], dtype=torch.int32, device=cuda)
        qr.qr_fm_count(fm, to_dev(pats.reshape(-1), cuda), None, k, d, pats.shape[0])
        torch.cuda.synchronize()
        if k < 9:
            assert int(to_host(d).astype(np.int64).sum()) == n - k + 1


@pytest.mark.parametrize("step,packed,refill", [(1, 1, 8), (2, 1, 8), (3, 1, 8), (3, 0, 8), (3, 1, 1), (3, 1, 32), (4, 1, 0)])
@pytest.mark.parametrize("bps", [2, 16, 64])
def test_fm_tuning_does_not_change_results(cuda, bps, step, packed, refill):
    torch = _torch()
    n = 90000
    w = gen.dna(31, n, 1)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    fm = qr.qr_fm_build(w, n)
    pats = mixed_patterns(np.random.default_rng(5), sym, 3000)
    cat, off, lens = oracle.pack_patterns(pats)
    ref = ora.count(cat, off, lens)
    L, m = 40, 5000
    fixed = gen.patterns(9, 1, m, L, w, n)
    ref_fixed = ora.count(fixed, np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32))
    qr.qr_set_tuning("fm_blocks_per_sm", bps)
    qr.qr_set_tuning("fm_step", step)
    qr.qr_set_tuning("fm_packed", packed)
    qr.qr_set_tuning("fm_refill", refill)
    try:
        d = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        qr.qr_fm_count(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, d, lens.size)
        d2 = torch.empty(m, dtype=torch.int32, device=cuda)
        work = torch.zeros(2, dtype=torch.uint64, device=cuda)
        qr.qr_fm_count_work(fm, to_dev(fixed, cuda), None, L, d2, m, work)
        torch.cuda.synchronize()
        db = torch.empty(m, dtype=torch.int32, device=cuda)
        dr = torch.empty(m, dtype=torch.int32, device=cuda)
        qr.qr_fm_count_both(fm, to_dev(fixed, cuda), None, L, db, dr, m)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("fm_blocks_per_sm", 64)
        qr.qr_set_tuning("fm_step", DEFAULT_FM_STEP)
        qr.qr_set_tuning("fm_packed", 1)
        qr.qr_set_tuning("fm_refill", 0)
    rc = np.concatenate([(3 - fixed[i * L:(i + 1) * L][::-1]).astype(np.uint8) for i in range(m)])
    assert np.array_equal(to_host(db).view(np.uint32), ref_fixed)
    assert np.array_equal(to_host(dr).view(np.uint32),
                          ora.count(rc, np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32)))
    assert np.array_equal(to_host(d).view(np.uint32), ref)
    assert np.array_equal(to_host(d2).view(np.uint32), ref_fixed)
    ts, tl = ora.work(fixed, np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32), skip=8, block=224)
    assert [int(x) for x in to_host(work)] == [ts, tl]


def revcomp(p):
    return (3 - np.asarray(p, np.uint8)[::-1]).astype(np.uint8)


def test_fm_count_both_strands(cuda):
    """qr_fm_count_both = counts of P and of RC(P), checked against the oracle
    counting explicitly reverse-complemented copies (RC([0,1]) = [2,3])."""
    torch = _torch()
    assert list(revcomp([0, 1])) == [2, 3]
    n = 150000
    w = gen.dna(61, n, 1)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    fm = qr.qr_fm_build(w, n)
    rng = np.random.default_rng(6)
    pats = mixed_patterns(rng, sym, 2000)
    pats += [revcomp(sym[a:a + 40]) for a in rng.integers(0, n - 40, 200)]
    cat, off, lens = oracle.pack_patterns(pats)
    rcat, roff, rlens = oracle.pack_patterns([revcomp(p) for p in pats])
    ref_f, ref_r = ora.count(cat, off, lens), ora.count(rcat, roff, rlens)
    assert ref_r[-200:].min() >= 1
    df = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    dr = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count_both(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, df, dr, lens.size)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(df).view(np.uint32), ref_f)
    assert np.array_equal(to_host(dr).view(np.uint32), ref_r)
    # fixed-length reads of the paper's shape (150 bp, 1% substitutions, either strand), host path
    L, m = 150, 3000
    reads = gen.patterns(7, 2, m, L, w, n)
    offs = np.arange(m, dtype=np.uint64) * L
    rr = np.concatenate([revcomp(reads[i * L:(i + 1) * L]) for i in range(m)])
    ref_f = ora.count(reads, offs, np.full(m, L, np.uint32))
    ref_r = ora.count(rr, offs, np.full(m, L, np.uint32))
    hf, hr = np.zeros(m, np.uint32), np.zeros(m, np.uint32)
    qr.qr_fm_count_both(fm, reads, None, L, hf, hr, m)
    qr.qr_sync()
    assert np.array_equal(hf, ref_f) and np.array_equal(hr, ref_r)
    assert (np.maximum(ref_f, ref_r) >= 1).mean() > 0.1          # error-free reads match one strand


@pytest.mark.parametrize("dyn", [0, 1])
@pytest.mark.parametrize("n,kind", [(1, 0), (30, 0), (1000, 0), (60000, 1), (131072 + 5, 0), ((1 << 20) + 7, 0)])
def test_fm_count_approx_one_mismatch(cuda, n, kind, dyn, fm_dyn_reset):
    """<=1-substitution counts (rank_4-driven branching + k-mer table variants; K = 8, and 10 at
    n >= 2^20) vs the oracle's direct Hamming-distance scan, static and dynamic pattern order;
    max_mismatches=0 equals exact counting."""
    torch = _torch()
    qr.qr_set_tuning("fm_dyn", dyn)
    w = gen.dna(71 + n, n, kind)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n)
    rng = np.random.default_rng(n)
    pats = mixed_patterns(rng, sym, 1200)
    for _ in range(200):                                   # exact and 1-/2-substitution variants
        L = int(rng.integers(1, 40)); a = int(rng.integers(0, max(1, n - L + 1)))
        p = sym[a:a + L].copy()
        for _s in range(int(rng.integers(0, 3))):
            if p.size:
                k = int(rng.integers(0, p.size)); p[k] = (p[k] + 1 + rng.integers(0, 3)) % 4
        pats.append(p)
    cat, off, lens = oracle.pack_patterns(pats)
    ref1 = oracle.scan_count_hd1(sym, cat, off, lens)
    ref0 = oracle.scan_count(sym, cat, off, lens)
    d1 = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    d0 = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count_approx(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, 1, d1, lens.size)
    qr.qr_fm_count_approx(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, 0, d0, lens.size)
    torch.cuda.synchronize()
    got1 = to_host(d1).view(np.uint32)
    bad = np.nonzero(got1 != ref1)[0]
    assert bad.size == 0, f"{bad.size} mismatches: {[(len(pats[i]), got1[i], ref1[i]) for i in bad[:5]]}"
    assert np.array_equal(to_host(d0).view(np.uint32), ref0)
    assert np.all(ref1 >= ref0)
    # fixed-length host path
    L, m = 24, 2000
    fx = gen.patterns(3, 1, m, L, w, n)
    h = np.zeros(m, np.uint32)
    qr.qr_fm_count_approx(fm, fx, None, L, 1, h, m)
    qr.qr_sync()
    assert np.array_equal(h, oracle.scan_count_hd1(sym, fx, np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32)))
    with pytest.raises(qr.QrError):
        qr.qr_fm_count_approx(fm, fx, None, L, 4, h, m)


@pytest.mark.parametrize("k", [0, 1, 5, 8, 10, 12, 13, 14])
def test_fm_kmer_width_does_not_change_counts(cuda, k):
    """Seeded vs unseeded counts are identical for every table width, incl. no table,
    on exact / both-strand / <=1-mismatch counting; the table holds the K-mer interval sizes."""
    torch = _torch()
    n = 70000
    w = gen.dna(81, n, 1)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, kmer_k=k)
    assert fm.kmer_k == k
    pats = mixed_patterns(np.random.default_rng(k), sym, 1500)
    cat, off, lens = oracle.pack_patterns(pats)
    ref = oracle.scan_count(sym, cat, off, lens)
    dc, dl = to_dev(cat, cuda), to_dev(lens, cuda)
    d = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count(fm, dc, dl, 0, d, lens.size)
    d1 = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count_approx(fm, dc, dl, 0, 1, d1, lens.size)
    df, dr = torch.empty_like(d), torch.empty_like(d)
    qr.qr_fm_count_both(fm, dc, dl, 0, df, dr, lens.size)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(d).view(np.uint32), ref)
    assert np.array_equal(to_host(df).view(np.uint32), ref)
    rcat, roff, rlens = oracle.pack_patterns([revcomp(p) for p in pats])
    assert np.array_equal(to_host(dr).view(np.uint32), oracle.scan_count(sym, rcat, roff, rlens))
    assert np.array_equal(to_host(d1).view(np.uint32), oracle.scan_count_hd1(sym, cat, off, lens))
    if 0 < k <= 8:
        t = qr.qr_fm_export_kmer(fm)
        assert t.shape == (4 ** k, 2)
        assert int((t[:, 1].astype(np.int64) - t[:, 0]).sum()) == n - k + 1


@pytest.mark.parametrize("step", [1, 2, 3, 4])
@pytest.mark.parametrize("fm_smem", [0, 1, 2])
def test_fm_superblock_source_does_not_change_results(cuda, fm_smem, step):
    """The count kernel's superblock words from global memory (0), from the raw array copied to
    shared memory (1, auto for small BWTs) or from the packed 8-per-u64 table in shared memory
    (2): a 3*10^6-symbol text spans 53 superblocks = 7 packed groups (odd: unequal halves), so
    every field of the packed encoding is read.  Exact + both strands, variable and fixed length."""
    torch = _torch()
    n = 3_000_000
    w = gen.dna(37, n, 0)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    fm = qr.qr_fm_build(w, n)
    pats = mixed_patterns(np.random.default_rng(7), sym, 4000)
    cat, off, lens = oracle.pack_patterns(pats)
    ref = ora.count(cat, off, lens)
    L, m = 48, 6000
    fixed = gen.patterns(10, 0, m, L, w, n)
    ref_fixed = ora.count(fixed, np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32))
    rc = np.concatenate([(3 - fixed[i * L:(i + 1) * L][::-1]).astype(np.uint8) for i in range(m)])
    ref_rc = ora.count(rc, np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32))
    qr.qr_set_tuning("fm_smem", fm_smem)
    qr.qr_set_tuning("fm_step", step)
    try:
        d = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        qr.qr_fm_count(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, d, lens.size)
        db = torch.empty(m, dtype=torch.int32, device=cuda)
        dr = torch.empty(m, dtype=torch.int32, device=cuda)
        qr.qr_fm_count_both(fm, to_dev(fixed, cuda), None, L, db, dr, m)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("fm_smem", 1)
        qr.qr_set_tuning("fm_step", DEFAULT_FM_STEP)
    assert np.array_equal(to_host(d).view(np.uint32), ref)
    assert np.array_equal(to_host(db).view(np.uint32), ref_fixed)
    assert np.array_equal(to_host(dr).view(np.uint32), ref_rc)


@pytest.mark.parametrize("dyn,seed", [(0, 0), (1, 1), (1, 2)])
@pytest.mark.parametrize("m", [1, 31, 63, 64, 65, 4097])
def test_fm_work_order_covers_every_task(cuda, dyn, seed, m):
    """Static grid-stride order (0) and the persistent warp-chunk order (1, default; seeds
    computed inline (fm_seed 1) or by the parallel pre-pass (2)) must count every pattern exactly
    once, for batch sizes around the chunk size (64) and the warp size, single strand and both
    strands (2m tasks), variable lengths."""
    torch = _torch()
    n = 120000
    w = gen.dna(41, n, 0)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    fm = qr.qr_fm_build(w, n)
    pats = mixed_patterns(np.random.default_rng(100 + m), sym, m)
    pats = pats[:m - 3] + pats[-3:] if m > 3 else pats[:m]   # keep whole-text / longer / empty
    cat, off, lens = oracle.pack_patterns(pats)
    assert lens.size == m
    ref = ora.count(cat, off, lens)
    rc_pats = [(3 - p[::-1]).astype(np.uint8) for p in pats]
    rcat, roff, rlens = oracle.pack_patterns(rc_pats)
    ref_rc = ora.count(rcat, roff, rlens)
    qr.qr_set_tuning("fm_dyn", dyn)
    qr.qr_set_tuning("fm_seed", seed)
    try:
        d = torch.full((m,), -1, dtype=torch.int32, device=cuda)
        qr.qr_fm_count(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, d, m)
        db = torch.full((m,), -1, dtype=torch.int32, device=cuda)
        dr = torch.full((m,), -1, dtype=torch.int32, device=cuda)
        qr.qr_fm_count_both(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, db, dr, m)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("fm_dyn", 1)
        qr.qr_set_tuning("fm_seed", 0)
    assert np.array_equal(to_host(d).view(np.uint32), ref)
    assert np.array_equal(to_host(db).view(np.uint32), ref)
    assert np.array_equal(to_host(dr).view(np.uint32), ref_rc)


def test_fm_default_kmer_width(cuda):
    """qr_fm_build's width: the paper's 8 below n = 2^20, 10 below 2^24, above 11 while the BWT
    layout + the 32 MiB 11-mer table fit in 60% of the L2 (126 MB on B200), else 12."""
    torch = _torch()
    for n, k in ((1000, 8), ((1 << 20) - 1, 8), (1 << 20, 10), ((1 << 24) - 1, 10), (1 << 24, 11), (1 << 26, 11),
                 (1 << 28, 12)):
        t = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=cuda)
        gen.dna_dev(50, n, 0, t)
        fm = qr.qr_fm_build(t, n)
        assert fm.kmer_k == k, (n, fm.kmer_k)
        fm.free()


@pytest.mark.parametrize("step", [0, 3])
@pytest.mark.parametrize("n,kind", [(1, 0), (7, 0), (100, 0), (1000, 0), (50000, 0), (25000, 1), (3_000_000, 0)])
@pytest.mark.parametrize("dyn", [0, 1])
def test_fm_over_quadrank16x2(cuda, n, kind, dyn, step, fm_dyn_reset):
    """QuadFm over the sector-local QuadRank16x2 BWT (qr_fm_build_opts): the k-mer table, exact
    counts (variable lengths, one and both strands), <= 1-substitution counts and the work
    instrumentation must equal the oracle / the QuadRank16-backed index, static and dynamic order."""
    torch = _torch()
    w = gen.dna(700 + n, n, kind)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    fm = qr.qr_fm_build(w, n, bwt_layout=qr.QR_LAYOUT_QUADRANK16X2)
    fm16 = qr.qr_fm_build(w, n)
    assert fm.kmer_k == fm16.kmer_k and fm.spos == ora.spos
    assert np.array_equal(qr.qr_fm_export_kmer(fm), qr.qr_fm_export_kmer(fm16))
    qr.qr_set_tuning("fm_dyn", dyn)
    qr.qr_set_tuning("fm_step", step)
    pats = mixed_patterns(np.random.default_rng(n), sym, 1500)
    cat, off, lens = oracle.pack_patterns(pats)
    ref = ora.count(cat, off, lens)
    d = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, d, lens.size)
    db = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    dr = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count_both(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, db, dr, lens.size)
    d1 = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count_approx(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, 1, d1, lens.size)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(d).view(np.uint32), ref)
    assert np.array_equal(to_host(db).view(np.uint32), ref)
    rc = [(3 - p[::-1]).astype(np.uint8) for p in pats]
    rcat, roff, rlens = oracle.pack_patterns(rc)
    assert np.array_equal(to_host(dr).view(np.uint32), ora.count(rcat, roff, rlens))
    if n <= 50000:
        assert np.array_equal(to_host(d1).view(np.uint32), oracle.scan_count_hd1(sym, cat, off, lens))
    else:
        d1b = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        qr.qr_fm_count_approx(fm16, to_dev(cat, cuda), to_dev(lens, cuda), 0, 1, d1b, lens.size)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(d1), to_host(d1b))
    if n >= 1000:
        L, m = 32, 3000
        fx = gen.patterns(11, 0, m, L, w, n)
        dw = torch.empty(m, dtype=torch.int32, device=cuda)
        work = torch.zeros(2, dtype=torch.uint64, device=cuda)
        qr.qr_fm_count_work(fm, to_dev(fx, cuda), None, L, dw, m, work)
        torch.cuda.synchronize()
        offs, lens_ = np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32)
        assert np.array_equal(to_host(dw).view(np.uint32), ora.count(fx, offs, lens_))
        # distinct 192-row lines (QuadRank16x2) per post-seed step, as the oracle counts them
        assert [int(x) for x in to_host(work)] == list(ora.work(fx, offs, lens_, skip=fm.kmer_k, block=192))


@pytest.mark.parametrize("kmax", [2, 3])
@pytest.mark.parametrize("bwt_layout", [None, qr.QR_LAYOUT_QUADRANK16X2])
@pytest.mark.parametrize("dyn", [0, 1])
@pytest.mark.parametrize("n,kind", [(1, 0), (40, 0), (3000, 0), (50000, 1), (131072 + 9, 0)])
def test_fm_count_approx_k_mismatches(cuda, n, kind, dyn, bwt_layout, kmax, fm_dyn_reset):
    """<=2 and <=3-substitution counts (rank_4 backtracking, one frame per mismatch level) vs the
    oracle's direct Hamming-distance scan, variable and fixed lengths, device and host pointers,
    both BWT layouts, static and dynamic pattern order; monotone in k."""
    torch = _torch()
    qr.qr_set_tuning("fm_dyn", dyn)
    w = gen.dna(91 + n, n, kind)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, bwt_layout=bwt_layout)
    rng = np.random.default_rng(n + kmax)
    pats = []
    for i in range(400):
        L = int(rng.integers(0, 13)) if i % 4 == 0 else int(rng.integers(1, 28))
        if i % 2 and n >= L:                               # substring with 0..4 substitutions
            a = int(rng.integers(0, max(1, n - L + 1)))
            p = sym[a:a + L].copy()
            for _s in range(int(rng.integers(0, 5))):
                if p.size:
                    k = int(rng.integers(0, p.size)); p[k] = (p[k] + 1 + rng.integers(0, 3)) % 4
        else:
            p = rng.integers(0, 4, L).astype(np.uint8)
        pats.append(p)
    pats.append(sym.copy())
    pats.append(np.concatenate([sym, sym[:2]]))
    cat, off, lens = oracle.pack_patterns(pats)
    ref = oracle.scan_count_hdk(sym, cat, off, lens, kmax)
    d = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count_approx(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, kmax, d, lens.size)
    torch.cuda.synchronize()
    got = to_host(d).view(np.uint32)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"{bad.size} mismatches: {[(len(pats[i]), got[i], ref[i]) for i in bad[:5]]}"
    assert np.all(ref >= oracle.scan_count_hdk(sym, cat, off, lens, kmax - 1))
    # fixed length, host pointers (staged path)
    L, m = 20, 300
    fx = np.concatenate([sym[a:a + L] if n >= L else rng.integers(0, 4, L).astype(np.uint8)
                         for a in rng.integers(0, max(1, n - L + 1), m)]).astype(np.uint8)
    if fx.size < m * L:
        fx = np.resize(fx, m * L)
    foff = np.arange(m, dtype=np.uint64) * L
    fref = oracle.scan_count_hdk(sym, fx, foff, np.full(m, L, np.uint32), kmax)
    h = np.zeros(m, np.uint32)
    qr.qr_fm_count_approx(fm, fx, None, L, kmax, h, m)
    qr.qr_sync()
    assert np.array_equal(h, fref)


def test_fm_count_approx_rejects_k_above_3(cuda):
    torch = _torch()
    w = gen.dna(5, 1000)
    fm = qr.qr_fm_build(w, 1000)
    d = torch.empty(4, dtype=torch.int32, device=cuda)
    pats = torch.zeros(4 * 8, dtype=torch.uint8, device=cuda)
    with pytest.raises(qr.QrError):
        qr.qr_fm_count_approx(fm, pats, None, 8, 4, d, 4)


def test_fm_host_variable_length_chunks(cuda):
    """Host-pointer batches with per-pattern lengths are staged in chunks of <= 2^22 patterns:
    a batch just over one chunk (forward and both strands) equals the oracle on every pattern."""
    n = 5000
    w = gen.dna(404, n)
    sym = gen.unpack_dna(w, n)
    ora = oracle.FmOracle(sym)
    rng = np.random.default_rng(404)
    m = (1 << 22) + 1003
    lens = rng.integers(0, 13, m).astype(np.uint32)
    cat = rng.integers(0, 4, int(lens.sum())).astype(np.uint8)
    off = np.concatenate([[0], np.cumsum(lens[:-1], dtype=np.uint64)]).astype(np.uint64)
    ref = ora.count(cat, off, lens)
    out = np.zeros(m, np.uint32)
    qr.qr_fm_count(fm := qr.qr_fm_build(w, n), cat, lens, 0, out, m)
    qr.qr_sync()
    assert np.array_equal(out, ref)
    rc_cat = np.concatenate([3 - cat[int(o):int(o) + int(L)][::-1] for o, L in zip(off[-2000:], lens[-2000:])])
    rc_off = np.concatenate([[0], np.cumsum(lens[-2000:][:-1], dtype=np.uint64)]).astype(np.uint64)
    of, orc = np.zeros(m, np.uint32), np.zeros(m, np.uint32)
    qr.qr_fm_count_both(fm, cat, lens, 0, of, orc, m)
    qr.qr_sync()
    assert np.array_equal(of, ref)
    assert np.array_equal(orc[-2000:], ora.count(rc_cat.astype(np.uint8), rc_off, lens[-2000:]))


@pytest.mark.parametrize("kmax", [0, 1, 2, 3])
@pytest.mark.parametrize("bwt_layout", [None, qr.QR_LAYOUT_QUADRANK16X2])
@pytest.mark.parametrize("n,kind", [(40, 0), (20000, 0), (60000, 1)])
def test_fm_count_approx_both_strands(cuda, n, kind, bwt_layout, kmax, fm_dyn_reset):
    """Both strands within k substitutions in one launch: forward counts equal the oracle's
    Hamming scan of P, reverse counts the scan of 3 - P reversed; device variable lengths, host
    fixed lengths (reads of the paper's shape), both work orders."""
    torch = _torch()
    w = gen.dna(505 + n, n, kind)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, bwt_layout=bwt_layout)
    rng = np.random.default_rng(n + kmax)
    pats = [rng.integers(0, 4, int(rng.integers(0, 26))).astype(np.uint8) for _ in range(150)]
    for _ in range(150):
        L = int(rng.integers(1, 26)); a = int(rng.integers(0, max(1, n - L + 1)))
        p = sym[a:a + L].copy()
        if rng.random() < 0.5:
            p = (3 - p[::-1]).astype(np.uint8)                 # a reverse-strand occurrence
        for _s in range(int(rng.integers(0, 3))):
            if p.size:
                k = int(rng.integers(0, p.size)); p[k] = (p[k] + 1 + rng.integers(0, 3)) % 4
        pats.append(p)
    rcs = [(3 - p[::-1]).astype(np.uint8) for p in pats]
    cat, off, lens = oracle.pack_patterns(pats)
    rcat, roff, rlens = oracle.pack_patterns(rcs)
    ref_f = oracle.scan_count_hdk(sym, cat, off, lens, kmax)
    ref_r = oracle.scan_count_hdk(sym, rcat, roff, rlens, kmax)
    for dyn in (0, 1):
        qr.qr_set_tuning("fm_dyn", dyn)
        df = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        dr = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        qr.qr_fm_count_approx_both(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, kmax, df, dr, lens.size)
        torch.cuda.synchronize()
        assert np.array_equal(to_host(df).view(np.uint32), ref_f), dyn
        assert np.array_equal(to_host(dr).view(np.uint32), ref_r), dyn
    L, m = 30, 200
    reads = gen.patterns(9, 2, m, L, w, n) if n > L else rng.integers(0, 4, m * L).astype(np.uint8)
    roffs = np.arange(m, dtype=np.uint64) * L
    rr = np.concatenate([3 - reads[i * L:(i + 1) * L][::-1] for i in range(m)]).astype(np.uint8)
    hf, hr = np.zeros(m, np.uint32), np.zeros(m, np.uint32)
    qr.qr_fm_count_approx_both(fm, reads, None, L, kmax, hf, hr, m)
    qr.qr_sync()
    assert np.array_equal(hf, oracle.scan_count_hdk(sym, reads, roffs, np.full(m, L, np.uint32), kmax))
    assert np.array_equal(hr, oracle.scan_count_hdk(sym, rr, roffs, np.full(m, L, np.uint32), kmax))


def test_fm_empty_batches(cuda):
    """m = 0 is a no-op (QR_OK, nothing written) for every FM entry point, device and host."""
    torch = _torch()
    w = gen.dna(77, 3000)
    fm = qr.qr_fm_build(w, 3000)
    d = torch.full((4,), 7, dtype=torch.int32, device=cuda)
    r = torch.full((4,), 7, dtype=torch.int32, device=cuda)
    p = torch.zeros(64, dtype=torch.uint8, device=cuda)
    qr.qr_fm_count(fm, p, None, 8, d, 0)
    qr.qr_fm_count_both(fm, p, None, 8, d, r, 0)
    for k in range(4):
        qr.qr_fm_count_approx(fm, p, None, 8, k, d, 0)
        qr.qr_fm_count_approx_both(fm, p, None, 8, k, d, r, 0)
    torch.cuda.synchronize()
    assert int(d.sum()) == 28 and int(r.sum()) == 28
    h = np.full(4, 7, np.uint32)
    qr.qr_fm_count(fm, np.zeros(64, np.uint8), np.zeros(4, np.uint32), 0, h, 0)
    qr.qr_sync()
    assert int(h.sum()) == 28


_ORA_CACHE = {}


@pytest.mark.parametrize("L", [12, 13, 43, 44, 45])
@pytest.mark.parametrize("strands", [1, 2])
def test_fm_packed_seed_boundaries(cuda, L, strands):
    """L2-resident count kernel with packed post-seed symbols (k_fm_seed_packed): a 2^24-symbol text
    takes K = 12, so L = 44 leaves exactly 32 symbols (the largest packed case), 45 falls back to
    the pattern window, 12 and 13 leave none and one.  Both strands, exact substrings and iid
    patterns, against the oracle's backward search."""
    torch = _torch()
    n = (1 << 24) + 77
    w = gen.dna(91, n, 0)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, kmer_k=12)
    assert fm.kmer_k == 12
    m = 6000
    fx = gen.patterns(92 + L, 0, m, L, w, n)
    offs, lens = np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32)
    d = torch.empty(m, dtype=torch.int32, device=cuda)
    dr = torch.empty(m, dtype=torch.int32, device=cuda)
    if strands == 1:
        qr.qr_fm_count(fm, to_dev(fx, cuda), None, L, d, m)
    else:
        qr.qr_fm_count_both(fm, to_dev(fx, cuda), None, L, d, dr, m)
    torch.cuda.synchronize()
    if n not in _ORA_CACHE:                               # one oracle SA for all parametrisations
        _ORA_CACHE[n] = oracle.FmOracle(sym)
    ora = _ORA_CACHE[n]
    sel = np.arange(0, m, 3)                              # the oracle on every third pattern
    cat = np.concatenate([fx[i * L:(i + 1) * L] for i in sel])
    so, sl = np.arange(sel.size, dtype=np.uint64) * L, np.full(sel.size, L, np.uint32)
    assert np.array_equal(to_host(d).view(np.uint32)[sel], ora.count(cat, so, sl))
    if strands == 2:
        rc = np.concatenate([revcomp(fx[i * L:(i + 1) * L]) for i in sel])
        assert np.array_equal(to_host(dr).view(np.uint32)[sel], ora.count(rc, so, sl))


@pytest.mark.parametrize("bwt_layout", [None, qr.QR_LAYOUT_QUADRANK16X2])
def test_fm_count_work_ex_accounting(cuda, bwt_layout):
    """qr_fm_count_work_ex (measurement counters of every count flavour): counts equal the plain
    calls'; exact one strand equals qr_fm_count_work and the oracle's post-seed steps / lines;
    both strands = forward + the reverse complements counted alone; approximate search counts at
    least the exact path's work and more lines than rank pairs; the counters do not depend on the
    work order (static / dynamic) — nor on the search order (breadth first, k = 1-3, or the
    recursive kernels)."""
    torch = _torch()
    n = 60000
    w = gen.dna(401, n, 1)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, bwt_layout=bwt_layout)
    ora = oracle.FmOracle(sym)
    L, m = 40, 3000
    fx = gen.patterns(402, 1, m, L, w, n)
    rcx = np.concatenate([revcomp(fx[i * L:(i + 1) * L]) for i in range(m)])
    offs, lens = np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32)
    block = 192 if bwt_layout else 224

    def work_of(pats, kmax, both, dyn=1):
        qr.qr_set_tuning("fm_dyn", dyn)
        o = torch.empty(m, dtype=torch.int32, device=cuda)
        orc = torch.empty(m, dtype=torch.int32, device=cuda) if both else None
        wk = torch.zeros(2, dtype=torch.uint64, device=cuda)
        qr.qr_fm_count_work_ex(fm, to_dev(pats, cuda), None, L, kmax, o, orc, m, wk)
        torch.cuda.synchronize()
        qr.qr_set_tuning("fm_dyn", 1)
        return [int(x) for x in to_host(wk)], to_host(o).view(np.uint32), None if orc is None else to_host(orc).view(np.uint32)

    (s1, l1), c1, _ = work_of(fx, 0, False)
    assert np.array_equal(c1, ora.count(fx, offs, lens))
    assert (s1, l1) == ora.work(fx, offs, lens, skip=fm.kmer_k, block=block)
    (sr, lr), cr, _ = work_of(rcx, 0, False)
    (sb, lb), cbf, cbr = work_of(fx, 0, True)
    assert (sb, lb) == (s1 + sr, l1 + lr)
    assert np.array_equal(cbf, c1) and np.array_equal(cbr, cr)
    for kmax in (1, 2, 3):
        (sa, la), ca, car = work_of(fx, kmax, True)        # breadth first (dynamic order) ...
        (sd, ld), _, _ = work_of(fx, kmax, True, dyn=0)    # ... and the recursive kernels count alike
        assert (sa, la) == (sd, ld)
        assert sa >= s1 + sr and la >= sa
        assert np.array_equal(ca, oracle.scan_count_hdk(sym, fx, offs, lens, kmax))
        assert np.array_equal(car, oracle.scan_count_hdk(sym, rcx, offs, lens, kmax))


def test_checksum_is_additive_over_shards(cuda):
    """qr_checksum (multi-GPU output verification): the checksum of a whole batch equals the sum
    mod 2^64 of its shards' checksums with global index offsets, for u64 and u32 outputs, and
    differs when one word or the index offset changes."""
    torch = _torch()
    rng = np.random.default_rng(3)
    for wb, dt in ((8, np.uint64), (4, np.uint32)):
        a = rng.integers(0, 2**63, 100003).astype(dt)
        d = to_dev(a, cuda)

        def cks(lo, hi, i0):
            acc = torch.zeros(1, dtype=torch.uint64, device=cuda)
            qr.qr_checksum(d[lo:hi], hi - lo, wb, i0, acc)
            torch.cuda.synchronize()
            return int(acc.view(torch.int64).item()) & (2**64 - 1)
        whole = cks(0, a.size, 0)
        parts = (cks(0, 777, 0) + cks(777, 50000, 777) + cks(50000, a.size, 50000)) & (2**64 - 1)
        assert whole == parts
        assert cks(0, a.size, 1) != whole
        b = a.copy()
        b[12345] ^= 1
        acc = torch.zeros(1, dtype=torch.uint64, device=cuda)
        qr.qr_checksum(to_dev(b, cuda), b.size, wb, 0, acc)
        torch.cuda.synchronize()
        assert int(acc.view(torch.int64).item()) & (2**64 - 1) != whole


def test_fm_default_width_dual_tables(cuda):
    """From n = 2^24 on a B200 the default build keeps an 11-mer table for the exact count and
    builds a 14-mer table for the approximate-search kernels on their first call; every count
    equals the oracle's and the single-table handles' (explicit widths 11 and 12), a clone made
    before the first approximate call builds its own, and four host threads on their own streams
    racing for a fresh handle's first approximate call all get exact counts."""
    torch = _torch()
    n = (1 << 24) + 5
    w = gen.dna(411, n, 0)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n)
    assert fm.kmer_k == 11
    L, m = 32, 300
    fx = gen.patterns(412, 0, m, L, w, n)
    offs, lens = np.arange(m, dtype=np.uint64) * L, np.full(m, L, np.uint32)
    handles = [fm, qr.qr_fm_build(w, n, kmer_k=11), qr.qr_fm_build(w, n, kmer_k=12), qr.qr_fm_clone_to_device(fm, 0)]
    refs = {kmax: oracle.scan_count_hdk(sym, fx, offs, lens, kmax) for kmax in (0, 1, 2)}
    for kmax in (0, 1, 2):
        for h in handles:
            d = torch.empty(m, dtype=torch.int32, device=cuda)
            qr.qr_fm_count_approx(h, to_dev(fx, cuda), None, L, kmax, d, m)
            torch.cuda.synchronize()
            assert np.array_equal(to_host(d).view(np.uint32), refs[kmax]), (kmax, h.kmer_k)
    import threading

    fresh = qr.qr_fm_build(w, n)
    errs, outs = [], {}

    def worker(i):
        try:
            s_ = torch.cuda.Stream()
            with torch.cuda.stream(s_):
                d = torch.empty(m, dtype=torch.int32, device=cuda)
                qr.qr_fm_count_approx(fresh, to_dev(fx, cuda), None, L, 1 + i % 2, d, m, s_)
                s_.synchronize()
                outs[i] = to_host(d).view(np.uint32)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t_ in ts:
        t_.start()
    for t_ in ts:
        t_.join()
    assert not errs, errs
    for i in range(4):
        assert np.array_equal(outs[i], refs[1 + i % 2]), i
    # a CUDA-graph capture of the first approximate call on a fresh handle: the wider table cannot
    # be built inside the capture, the captured call uses the count's table and is exact
    fresh2 = qr.qr_fm_build(w, n)
    dp = to_dev(fx, cuda)
    dg = torch.empty(m, dtype=torch.int32, device=cuda)
    s2 = torch.cuda.Stream()
    s2.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s2):
        qr.qr_fm_count_approx(fresh2, dp, None, L, 2, dg, m, stream=torch.cuda.current_stream())
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(to_host(dg).view(np.uint32), refs[2])


@pytest.mark.parametrize("bwt_layout", [None, qr.QR_LAYOUT_QUADRANK16X2])
@pytest.mark.parametrize("dyn", [0, 1])
@pytest.mark.parametrize("n,kind", [(1, 0), (57, 0), (5000, 0), (60000, 1), (300000, 0)])
def test_fm_approx_all_k_both_strands(cuda, bwt_layout, dyn, n, kind):
    """Approximate search for k = 1, 2, 3 on both strands in one launch, variable lengths (empty,
    shorter than the table width, longer), static and dynamic order, against the oracle's direct
    scan (the k >= 2 kernel keeps its backtracking frames in shared memory, FmFrames)."""
    torch = _torch()
    w = gen.dna(900 + n, n, kind)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, bwt_layout=bwt_layout)
    rng = np.random.default_rng(n)
    pats = mixed_patterns(rng, sym, 160)
    cat, off, lens = oracle.pack_patterns(pats)
    rc = [revcomp(p) for p in pats]
    rcat, roff, rlens = oracle.pack_patterns(rc)
    qr.qr_set_tuning("fm_dyn", dyn)
    try:
        for kmax in (1, 2, 3):
            df = torch.empty(lens.size, dtype=torch.int32, device=cuda)
            dr = torch.empty(lens.size, dtype=torch.int32, device=cuda)
            qr.qr_fm_count_approx_both(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, kmax, df, dr, lens.size)
            torch.cuda.synchronize()
            assert np.array_equal(to_host(df).view(np.uint32), oracle.scan_count_hdk(sym, cat, off, lens, kmax)), kmax
            assert np.array_equal(to_host(dr).view(np.uint32), oracle.scan_count_hdk(sym, rcat, roff, rlens, kmax)), kmax
    finally:
        qr.qr_set_tuning("fm_dyn", 1)


@pytest.mark.parametrize("n,kind,kmer_k", [(5000, 0, None), (300000, 1, 8), (300000, 0, 12)])
def test_fm_approx_presence_bitmap(cuda, n, kind, kmer_k):
    """The approximate search's k-mer presence bitmap (fm_kbits: 0 auto = sparse tables only,
    1 never, 2 always) changes no count: k = 1, 2, 3 on both strands against the oracle with the
    bitmap off, forced on (also over a dense table, n = 300000 at K = 8) and auto, switched back
    and forth on one handle (built on first use, kept for later calls)."""
    torch = _torch()
    w = gen.dna(1300 + n, n, kind)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, kmer_k=kmer_k) if kmer_k else qr.qr_fm_build(w, n)
    rng = np.random.default_rng(n + 7)
    pats = mixed_patterns(rng, sym, 120)
    cat, off, lens = oracle.pack_patterns(pats)
    rc = [revcomp(p) for p in pats]
    rcat, roff, rlens = oracle.pack_patterns(rc)
    refs = {k: (oracle.scan_count_hdk(sym, cat, off, lens, k), oracle.scan_count_hdk(sym, rcat, roff, rlens, k))
            for k in (1, 2, 3)}
    dp, dl = to_dev(cat, cuda), to_dev(lens, cuda)
    try:
        for knob in (1, 2, 0, 1, 2):
            qr.qr_set_tuning("fm_kbits", knob)
            for kmax in (1, 2, 3):
                df = torch.empty(lens.size, dtype=torch.int32, device=cuda)
                dr = torch.empty(lens.size, dtype=torch.int32, device=cuda)
                qr.qr_fm_count_approx_both(fm, dp, dl, 0, kmax, df, dr, lens.size)
                torch.cuda.synchronize()
                assert np.array_equal(to_host(df).view(np.uint32), refs[kmax][0]), (knob, kmax)
                assert np.array_equal(to_host(dr).view(np.uint32), refs[kmax][1]), (knob, kmax)
    finally:
        qr.qr_set_tuning("fm_kbits", 0)


@pytest.mark.parametrize("space", ["host", "device"])
def test_fm_build_from_bytes(cuda, space):
    """qr_fm_build_u8 (one byte per symbol, SURVEY §8(b)'s input form, packed on the GPU) builds
    the same index as qr_fm_build from 2-bit words: same spos, C, k-mer table and counts (vs the
    oracle); a byte > 3 is QR_EINVAL."""
    torch = _torch()
    n = 70001
    w = gen.dna(431, n, 1)
    sym = gen.unpack_dna(w, n)
    src = sym if space == "host" else to_dev(sym, cuda)
    fb = qr.qr_fm_build_u8(src, n)
    fw = qr.qr_fm_build(w, n)
    assert (fb.spos, fb.C, fb.kmer_k) == (fw.spos, fw.C, fw.kmer_k)
    assert np.array_equal(qr.qr_fm_export_kmer(fb), qr.qr_fm_export_kmer(fw))
    pats = mixed_patterns(np.random.default_rng(3), sym, 500)
    cat, off, lens = oracle.pack_patterns(pats)
    d = torch.empty(lens.size, dtype=torch.int32, device=cuda)
    qr.qr_fm_count(fb, to_dev(cat, cuda), to_dev(lens, cuda), 0, d, lens.size)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(d).view(np.uint32), oracle.FmOracle(sym).count(cat, off, lens))
    bad = sym.copy()
    bad[n // 2] = 4
    with pytest.raises(qr.QrError) as e:
        qr.qr_fm_build_u8(bad if space == "host" else to_dev(bad, cuda), n)
    assert e.value.status == qr.QR_EINVAL


@pytest.mark.parametrize("bwt_layout", [None, qr.QR_LAYOUT_QUADRANK16X2])
@pytest.mark.parametrize("queue", [0, 1, 4])
@pytest.mark.parametrize("bfs,kbits", [(0, 0), (2, 1), (2, 2)])
@pytest.mark.parametrize("kmax", [1, 2])
def test_fm_approx_breadth_first_queues(cuda, bwt_layout, queue, bfs, kbits, kmax, fm_dyn_reset):
    """k = 1, 2 breadth first (seed items, the paths' branch items, their continuations) with
    the interval queues sized 0 (every branch searched inline by its lane), 1 or 4 items per task,
    with and without the presence bitmap, against the recursive kernel's oracle — the direct
    Hamming scan — on both strands, ragged lengths (shorter than, equal to and longer than the
    seed width)."""
    torch = _torch()
    n = 300_007
    w = gen.dna(401, n, 0)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, bwt_layout=bwt_layout)
    rng = np.random.default_rng(7)
    pats = []
    for i in range(3000):
        L = int(rng.integers(1, 60))
        a = int(rng.integers(0, n - L))
        p = sym[a:a + L].copy()
        if i % 3 and L:
            k = int(rng.integers(0, L)); p[k] = (p[k] + 1 + rng.integers(0, 3)) % 4
        pats.append(p)
    cat, off, lens = oracle.pack_patterns(pats)
    hd = oracle.scan_count_hd1 if kmax == 1 else (lambda *a: oracle.scan_count_hdk(*a, 2))
    ref = hd(sym, cat, off, lens)
    ccat, coff, clens = oracle.pack_patterns([revcomp(p) for p in pats])
    ref_rc = hd(sym, ccat, coff, clens)
    try:
        qr.qr_set_tuning("fm_ax_bfs", bfs)
        qr.qr_set_tuning("fm_ax_queue", queue)
        qr.qr_set_tuning("fm_kbits", kbits)
        df = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        dr = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        qr.qr_fm_count_approx_both(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, kmax, df, dr, lens.size)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("fm_ax_bfs", 1)
        qr.qr_set_tuning("fm_ax_queue", 4)
        qr.qr_set_tuning("fm_kbits", 0)
    assert np.array_equal(to_host(df).view(np.uint32), ref)
    assert np.array_equal(to_host(dr).view(np.uint32), ref_rc)


@pytest.mark.parametrize("bwt_layout", [None, qr.QR_LAYOUT_QUADRANK16X2])
@pytest.mark.parametrize("L", [10, 24, 33])
@pytest.mark.parametrize("queue", [0, 4])
def test_fm_approx3_breadth_first_fixed_length(cuda, bwt_layout, L, queue, fm_dyn_reset):
    """k = 3 breadth first (fixed-length batches: the level-2 queue holds 3 (L - K) items per
    task) against the recursive kernel and the oracle's Hamming scan, both strands; L = 10 is the
    table width (every variant a leaf), with the level-1 and level-0 queues sized 0 and 4."""
    torch = _torch()
    n = 200_003
    w = gen.dna(403, n, 0)
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n, kmer_k=10, bwt_layout=bwt_layout)
    m = 600
    pats = gen.patterns(11, 1, m, L, w, n)              # substrings with 0-2 substitutions
    offs = np.arange(m, dtype=np.uint64) * L
    lens = np.full(m, L, np.uint32)
    ref = oracle.scan_count_hdk(sym, pats, offs, lens, 3)
    rc = np.concatenate([revcomp(pats[i * L:(i + 1) * L]) for i in range(m)])
    ref_rc = oracle.scan_count_hdk(sym, rc, offs, lens, 3)
    got = {}
    try:
        qr.qr_set_tuning("fm_ax_queue", queue)
        for bfs in (0, 2):
            qr.qr_set_tuning("fm_ax_bfs", bfs)
            df = torch.empty(m, dtype=torch.int32, device=cuda)
            dr = torch.empty(m, dtype=torch.int32, device=cuda)
            qr.qr_fm_count_approx_both(fm, to_dev(pats, cuda), None, L, 3, df, dr, m)
            torch.cuda.synchronize()
            got[bfs] = (to_host(df).view(np.uint32), to_host(dr).view(np.uint32))
    finally:
        qr.qr_set_tuning("fm_ax_bfs", 1)
        qr.qr_set_tuning("fm_ax_queue", 4)
    for bfs in (0, 2):
        assert np.array_equal(got[bfs][0], ref), bfs
        assert np.array_equal(got[bfs][1], ref_rc), bfs
