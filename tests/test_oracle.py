"""Pins for the CPU oracle (oracle/oracle.c) and the seeded generators (gen/).

Each test checks the oracle against something other than itself: brute-force
sums written with numpy primitives, closed forms, invariants, special cases, an
independent Python re-implementation (suffix sort by comparison, substring
scan), and the worked example of SPEC.md:329 (tests/golden/).
"""
import itertools
import json
import os

import numpy as np
import pytest

import gen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def unpack_bits(words, n):
    b = np.unpackbits(words.view(np.uint8), bitorder="little")
    return b[:n].astype(np.int64)


def brute_rank_bits(words, n):
    """rank(q) for every q in [0, n] as a cumulative sum."""
    return np.concatenate([[0], np.cumsum(unpack_bits(words, n))]).astype(np.uint64)


def unpack_dna_np(words, n):
    b = words.view(np.uint8)
    sym = np.stack([(b >> (2 * k)) & 3 for k in range(4)], axis=1).reshape(-1)
    return sym[:n].astype(np.int64)


def brute_rank_dna(sym):
    """rank(q, c) for all q in [0,n], c in 0..3."""
    onehot = (sym[:, None] == np.arange(4)[None, :]).astype(np.int64)
    return np.vstack([np.zeros((1, 4), np.int64), np.cumsum(onehot, axis=0)]).astype(np.uint64)


# ----------------------------------------------------------------- generators
def _py_hash(seed, tag, i):
    M = (1 << 64) - 1
    z = ((seed ^ (tag * 0xD1B54A32D192ED03 & M)) + (i + 1) * 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_gen_matches_python_reimplementation():
    w = gen.bits(7, 64 * 5 + 13)
    for k in range(5):
        assert int(w[k]) == _py_hash(7, 1, k)
    assert int(w[5]) == _py_hash(7, 1, 5) & ((1 << 13) - 1)          # tail masked
    q = gen.queries(3, 1000, 50, i0=10)
    for k in range(50):
        assert int(q[k]) == (_py_hash(3, 3, 10 + k) * 1001) >> 64
    _, c = gen.queries(3, 1000, 20, with_c=True)
    assert [int(x) for x in c] == [_py_hash(3, 4, k) & 3 for k in range(20)]
    d = gen.dna(5, 40)
    assert int(d[0]) == _py_hash(5, 2, 0)
    assert int(d[1]) == _py_hash(5, 2, 1) & ((1 << 16) - 1)
    pb = gen.bits(9, 64, p=0.01)
    thr = int(0.01 * 2.0**64)
    assert int(pb[0]) == sum(1 << b for b in range(64) if _py_hash(9, 1, b) < thr)


def test_gen_determinism_and_uniformity():
    a = gen.dna(11, 1 << 20)
    assert np.array_equal(a, gen.dna(11, 1 << 20))
    assert not np.array_equal(a, gen.dna(12, 1 << 20))
    sym = unpack_dna_np(a, 1 << 20)
    cnt = np.bincount(sym, minlength=4)
    exp = (1 << 20) / 4
    chi2 = ((cnt - exp) ** 2 / exp).sum()
    assert chi2 < 30  # 3 dof; p ~ 1e-6
    b = gen.bits(13, 1 << 22, p=0.01)
    ones = unpack_bits(b, 1 << 22).sum()
    assert abs(ones - 0.01 * (1 << 22)) < 6 * np.sqrt(0.01 * (1 << 22))
    q = gen.queries(1, 10**6, 10**5)
    assert q.max() <= 10**6 and q.min() >= 0


def test_gen_block_repeat_text_structure():
    n = 5 * gen.BLOCK + 777
    sym = gen.unpack_dna(gen.dna(21, n, kind=1), n)
    assert sym.max() <= 3 and len(sym) == n
    # a copied block differs from its source in about 1% of positions
    blocks = [sym[i * gen.BLOCK:(i + 1) * gen.BLOCK] for i in range(5)]
    best = min(np.mean(blocks[b] != blocks[s]) for b in range(1, 5) for s in range(b))
    big = gen.unpack_dna(gen.dna(21, 60 * gen.BLOCK, kind=1), 60 * gen.BLOCK)
    bl = [big[i * gen.BLOCK:(i + 1) * gen.BLOCK] for i in range(60)]
    copies = sum(1 for b in range(1, 60) if min(np.mean(bl[b] != bl[s]) for s in range(b)) < 0.05)
    assert 8 <= copies <= 30        # ~0.3 * 59
    assert best >= 0.0


def test_gen_patterns_recipe():
    n = 10000
    text = gen.dna(4, n)
    sym = gen.unpack_dna(text, n)
    pats = gen.patterns(4, 0, 10, 32, text, n).reshape(10, 32)
    for i in range(0, 10, 2):
        pos = (_py_hash(4, 9, i) * (n - 32 + 1)) >> 64
        assert np.array_equal(pats[i], sym[pos:pos + 32])
    rd = gen.patterns(4, 2, 40, 150, text, n).reshape(40, 150)
    pm = 0x028F5C28F5C28F5C                                      # QRG_P_MUT = floor(0.01 * 2^64)
    for i in range(40):
        pos = (_py_hash(4, 9, i) * (n - 150 + 1)) >> 64
        exp = sym[pos:pos + 150].copy()
        for k in range(150):
            if _py_hash(4, 13, i * 150 + k) < pm:
                exp[k] = (exp[k] + 1 + ((_py_hash(4, 14, i * 150 + k) * 3) >> 64)) & 3
        if _py_hash(4, 15, i) & 1:
            exp = (3 - exp[::-1]).astype(np.uint8)
        assert np.array_equal(rd[i], exp)
    p5 = gen.patterns(4, 1, 30, 100, text, n).reshape(30, 100)
    for i in range(30):
        pos = (_py_hash(4, 9, i) * (n - 100 + 1)) >> 64
        s = (_py_hash(4, 11, i) * 3) >> 64
        assert int((p5[i] != sym[pos:pos + 100]).sum()) == s


# ----------------------------------------------------------------- rank sigma=2
@pytest.mark.parametrize("n", [0, 1, 2, 63, 64, 65, 127, 128, 495, 496, 497, 992, 1000, 2000])
@pytest.mark.parametrize("p", [0.5, 0.01, 1.0])
def test_rank_bits_bruteforce_every_q(n, p):
    w = gen.bits(100 + n, n, p)
    o = oracle.BitsOracle(w, n)
    q = np.arange(n + 1, dtype=np.uint64)
    r = o.rank(q)
    ref = brute_rank_bits(w, n)
    assert np.array_equal(r, ref)
    assert r[0] == 0                                       # rank(0) = 0
    assert r[-1] == unpack_bits(w, n).sum()                # rank(n) = total
    assert np.array_equal(np.diff(r.astype(np.int64)), unpack_bits(w, n))   # increments = t_q
    if p == 1.0:
        assert np.array_equal(r, q)                        # all-ones: rank(q) = q
    r0 = o.rank(q, np.zeros(n + 1, np.uint8))
    assert np.array_equal(r0, q - r)                       # rank(q,0) = q - rank(q,1)


def test_rank_bits_all_zero_and_random_sizes():
    rng = np.random.default_rng(0)
    for n in rng.integers(1, 1 << 16, size=6):
        n = int(n)
        w = np.zeros((n + 63) // 64, np.uint64)
        assert not oracle.BitsOracle(w, n).rank(np.arange(n + 1, dtype=np.uint64)).any()
        w = gen.bits(int(n), n)
        assert np.array_equal(oracle.BitsOracle(w, n).rank(np.arange(n + 1, dtype=np.uint64)), brute_rank_bits(w, n))


# ----------------------------------------------------------------- rank sigma=4
@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 95, 96, 97, 223, 224, 225, 448, 1000, 3001])
def test_rank_dna_bruteforce_every_q(n):
    w = gen.dna(200 + n, n)
    o = oracle.DnaOracle(w, n)
    sym = unpack_dna_np(w, n)
    ref = brute_rank_dna(sym)
    q = np.repeat(np.arange(n + 1, dtype=np.uint64), 4)
    c = np.tile(np.arange(4, dtype=np.uint8), n + 1)
    r = o.rank(q, c).reshape(n + 1, 4)
    assert np.array_equal(r, ref)
    a4 = o.rank_all4(np.arange(n + 1, dtype=np.uint64))
    assert np.array_equal(a4, ref)
    assert np.array_equal(a4.sum(axis=1), np.arange(n + 1, dtype=np.uint64))   # sum_c rank(q,c) = q
    assert np.array_equal(a4[-1], np.bincount(sym, minlength=4).astype(np.uint64))


def test_rank_dna_all_G():
    n = 1000
    w = np.full((n + 31) // 32, 0xAAAAAAAAAAAAAAAA, np.uint64)     # every char = G (2)
    w[-1] &= (1 << (2 * (n % 32))) - 1
    a4 = oracle.DnaOracle(w, n).rank_all4(np.arange(n + 1, dtype=np.uint64))
    q = np.arange(n + 1, dtype=np.uint64)
    assert np.array_equal(a4, np.stack([0 * q, 0 * q, q, 0 * q], axis=1))


# ----------------------------------------------------------------- suffix array / BWT
def naive_sa(sym):
    s = list(sym)
    return sorted(range(len(s) + 1), key=lambda i: s[i:] + [-1])


def test_sa_golden_acgt():
    g = json.load(open(os.path.join(GOLDEN, "spec_acgt_example.json")))
    f = oracle.FmOracle(np.array(g["text"], np.uint8))
    assert list(f.sa) == g["sa"]
    assert list(f.bwt) == g["bwt_symbols_dollar_is_4"]
    assert f.spos == g["spos"]
    assert list(f.C) == g["C_ACGT_then_N"]


@pytest.mark.parametrize("kind", ["random", "allA", "periodic", "tiny"])
def test_sa_vs_naive_comparison_sort(kind):
    rng = np.random.default_rng(5)
    for t in range(20):
        if kind == "random":
            s = rng.integers(0, 4, size=int(rng.integers(1, 300)))
        elif kind == "allA":
            s = np.zeros(int(rng.integers(1, 200)), np.int64)
        elif kind == "periodic":
            per = rng.integers(0, 4, size=int(rng.integers(1, 6)))
            s = np.tile(per, 50)[: int(rng.integers(1, 250))]
        else:
            s = rng.integers(0, 4, size=int(rng.integers(1, 4)))
        sa = oracle.suffix_array(s.astype(np.uint8))
        assert list(sa) == naive_sa(s.tolist())


# ----------------------------------------------------------------- FM count
def brute_count(sym, pat):
    s = sym.tolist(); p = list(pat)
    if len(p) == 0:
        return len(s) + 1
    return sum(1 for i in range(len(s) - len(p) + 1) if s[i:i + len(p)] == p)


def test_fm_counts_vs_bruteforce_small_texts():
    rng = np.random.default_rng(9)
    for t in range(25):
        n = int(rng.integers(1, 400))
        sym = rng.integers(0, 4, size=n).astype(np.uint8) if t % 3 else np.tile(rng.integers(0, 4, 3), 200)[:n].astype(np.uint8)
        f = oracle.FmOracle(sym)
        pats = [rng.integers(0, 4, size=int(rng.integers(0, 9))).astype(np.uint8) for _ in range(40)]
        for _ in range(20):                               # exact substrings
            a = int(rng.integers(0, n)); L = int(rng.integers(1, 12))
            pats.append(sym[a:a + L].copy())
        cat, off, lens = oracle.pack_patterns(pats)
        ref = np.array([brute_count(sym, p) for p in pats], np.uint32)
        assert np.array_equal(f.count(cat, off, lens), ref)
        assert np.array_equal(f.sa_count(cat, off, lens), ref)
        assert np.array_equal(oracle.scan_count(sym, cat, off, lens), ref)


def test_fm_special_cases():
    f = oracle.FmOracle(np.zeros(3, np.uint8))                   # "AAA"
    cat, off, lens = oracle.pack_patterns([np.array([0, 0], np.uint8), np.array([0, 0, 0, 0], np.uint8),
                                           np.zeros(0, np.uint8), np.array([1], np.uint8)])
    assert list(f.count(cat, off, lens)) == [2, 0, 4, 0]        # overlapping; longer than text; empty = n+1


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_fm_kmer_partition_identity(k):
    n = 3000
    sym = gen.unpack_dna(gen.dna(77, n), n)
    f = oracle.FmOracle(sym)
    pats = [np.array(p, np.uint8) for p in itertools.product(range(4), repeat=k)]
    cat, off, lens = oracle.pack_patterns(pats)
    cnt = f.count(cat, off, lens)
    assert int(cnt.sum()) == n - k + 1                            # every k-window counted once
    if k <= 3:
        assert np.array_equal(cnt, np.array([brute_count(sym, p) for p in pats], np.uint32))


def test_fm_work_instrumentation_consistent():
    n = 5000
    sym = gen.unpack_dna(gen.dna(3, n), n)
    text = gen.dna(3, n)
    f = oracle.FmOracle(sym)
    cat = gen.patterns(3, 0, 200, 32, text, n)
    off = np.arange(200, dtype=np.uint64) * 32
    lens = np.full(200, 32, np.uint32)
    cnt, steps = f.count(cat, off, lens, with_steps=True)
    ts, tl = f.work(cat, off, lens, skip=0, block=224)
    assert ts == int(steps.sum())
    assert ts <= tl <= 2 * ts
    assert np.array_equal(cnt[0::2] >= 1, np.ones(100, bool))    # exact substrings occur


def _suffixes(sym):
    """Every suffix of T$ as a tuple, '$' = -1 (smaller than every symbol)."""
    return [tuple(int(x) for x in sym[i:]) + (-1,) for i in range(len(sym) + 1)]


def _brute_interval(suf, Q):
    """[lo, hi) of Q in the sorted suffixes of T$, from the suffix strings themselves
    (no BWT, no LF mapping): lo = #suffixes whose first |Q| symbols compare below Q
    ('$' = -1, smaller than every symbol), hi = lo + #suffixes that start with Q
    (App. D: a BWT interval is the block of rows prefixed by Q)."""
    L = len(Q)
    Qt = tuple(int(x) for x in Q)
    lo = cnt = 0
    for s_i in suf:
        head = s_i[:L]
        if head < Qt:
            lo += 1
        elif head == Qt:
            cnt += 1
    return lo, lo + cnt


def _brute_work(sym, suf, P, skip, block):
    """(post-seed backward steps, distinct `block`-row lines touched) for one pattern,
    derived from the definition of backward search: the step that
    consumes P[j] runs iff the interval of P[j+1:] is non-empty (counted by a direct scan
    of the text), it ranks at that interval's lo and hi, and the first `skip` steps of a
    pattern of >= skip symbols are seeded by the k-mer table and not counted."""
    L = len(P)
    sk = skip if L >= skip else 0
    steps = lines = 0
    for t, j in enumerate(range(L - 1, -1, -1)):
        Q = P[j + 1:]
        occ = len(sym) + 1 if len(Q) == 0 else sum(
            1 for a in range(len(sym) - len(Q) + 1) if np.array_equal(sym[a:a + len(Q)], Q))
        if occ == 0:
            break
        if t >= sk:
            lo, hi = _brute_interval(suf, Q)
            assert hi - lo == occ                     # the two brute-force views agree
            steps += 1
            lines += 1 if lo // block == hi // block else 2
    return steps, lines


@pytest.mark.parametrize("block", [224, 192, 64, 7])
def test_fm_work_vs_bruteforce_intervals(block):
    """Pin for or_fm_work (SURVEY.md §8(c) instrumented mode, the FM algorithmic-bytes
    denominator): per pattern, recompute the executed post-seed steps and the distinct lines
    from brute-force suffix intervals, never from the oracle's own loop.  Covers patterns
    shorter than the skip, intervals that empty mid-pattern, exact substrings (never empty),
    repetitive texts (wide intervals that straddle lines) and skip = 0."""
    rng = np.random.default_rng(block)
    for t in range(6):
        n = int(rng.integers(40, 300))
        if t % 3 == 0:
            sym = rng.integers(0, 4, n).astype(np.uint8)
        elif t % 3 == 1:
            sym = np.tile(rng.integers(0, 4, 3), n)[:n].astype(np.uint8)
        else:
            sym = np.where(rng.random(n) < 0.9, 0, rng.integers(0, 4, n)).astype(np.uint8)
        f = oracle.FmOracle(sym)
        suf = _suffixes(sym)
        pats = [rng.integers(0, 4, int(rng.integers(0, 12))).astype(np.uint8) for _ in range(12)]
        pats += [sym[a:a + int(rng.integers(1, 20))].copy() for a in rng.integers(0, n, 8)]
        # exact substring with one late substitution: the interval empties mid-pattern
        for a in rng.integers(0, max(1, n - 16), 4):
            p = sym[a:a + 16].copy()
            if p.size:
                p[1] = (p[1] + 1) % 4
            pats.append(p)
        for skip in (0, 3, 8):
            exp_s = exp_l = 0
            for p in pats:
                s_, l_ = _brute_work(sym, suf, p, skip, block)
                exp_s += s_
                exp_l += l_
                cat1, off1, len1 = oracle.pack_patterns([p])
                assert f.work(cat1, off1, len1, skip=skip, block=block) == (s_, l_), (list(p), skip)
            cat, off, lens = oracle.pack_patterns(pats)
            assert f.work(cat, off, lens, skip=skip, block=block) == (exp_s, exp_l)


def test_hd1_scan_vs_bruteforce_and_variant_sum():
    """<=1-substitution counts: Python brute force on tiny texts, and the identity
    count_hd1(P) = sum over P and its 3L single-substitution variants of the exact count."""
    rng = np.random.default_rng(12)
    for t in range(12):
        n = int(rng.integers(1, 300))
        sym = rng.integers(0, 4, n).astype(np.uint8) if t % 2 else np.tile(rng.integers(0, 4, 2), 200)[:n].astype(np.uint8)
        f = oracle.FmOracle(sym)
        pats = [rng.integers(0, 4, int(rng.integers(0, 10))).astype(np.uint8) for _ in range(25)]
        pats += [sym[a:a + 6].copy() for a in rng.integers(0, n, 10)]
        cat, off, lens = oracle.pack_patterns(pats)
        got = oracle.scan_count_hd1(sym, cat, off, lens)
        for p, g in zip(pats, got):
            L = len(p)
            if L == 0:
                assert g == n + 1
                continue
            brute = sum(1 for i in range(n - L + 1) if int((sym[i:i + L] != p).sum()) <= 1)
            assert g == brute
            variants = [p] + [np.concatenate([p[:j], [(p[j] + d) % 4], p[j + 1:]]).astype(np.uint8)
                              for j in range(L) for d in (1, 2, 3)]
            vc, vo, vl = oracle.pack_patterns(variants)
            assert int(f.count(vc, vo, vl).astype(np.int64).sum()) == g


def test_hdk_scan_pins():
    """<=k-substitution counts (k = 0..3): Python brute force on tiny texts; k = 0 and 1 agree
    with the exact scan and the <=1 scan; k >= L counts every position; and the identity
    count_hdk(P) = sum of the exact counts (backward search over the simple BWT) of every string
    within Hamming distance k of P, enumerated over all 4^L strings for L <= 5."""
    import itertools

    rng = np.random.default_rng(31)
    for t in range(10):
        n = int(rng.integers(1, 260))
        sym = rng.integers(0, 4, n).astype(np.uint8) if t % 2 else np.tile(rng.integers(0, 4, 3), 100)[:n].astype(np.uint8)
        f = oracle.FmOracle(sym)
        pats = [rng.integers(0, 4, int(rng.integers(0, 9))).astype(np.uint8) for _ in range(14)]
        pats += [sym[a:a + 5].copy() for a in rng.integers(0, n, 6)]
        cat, off, lens = oracle.pack_patterns(pats)
        by_k = {k: oracle.scan_count_hdk(sym, cat, off, lens, k) for k in range(4)}
        assert np.array_equal(by_k[0], oracle.scan_count(sym, cat, off, lens))
        assert np.array_equal(by_k[1], oracle.scan_count_hd1(sym, cat, off, lens))
        for i, p in enumerate(pats):
            L = len(p)
            for k in range(4):
                g = int(by_k[k][i])
                if L == 0:
                    assert g == n + 1
                    continue
                brute = sum(1 for a in range(n - L + 1) if int((sym[a:a + L] != p).sum()) <= k)
                assert g == brute
                if k >= L:
                    assert g == max(0, n - L + 1)
                if k >= 2 and L <= 5:
                    near = [np.array(v, np.uint8) for v in itertools.product(range(4), repeat=L)
                            if sum(int(a != b) for a, b in zip(v, p)) <= k]
                    vc, vo, vl = oracle.pack_patterns(near)
                    assert int(f.count(vc, vo, vl).astype(np.int64).sum()) == g
            assert all(by_k[k][i] <= by_k[k + 1][i] for k in range(3))


def test_scan_count_bucketed_equals_direct_scan():
    """or_scan_count_bucketed (the configs[4] full-size check's counter) against the plain direct
    scan and Python brute force: random and repetitive texts, patterns of 0..40 symbols (both sides
    of the 8-symbol bucket key), exact substrings, substituted ones, longer than the text."""
    rng = np.random.default_rng(77)
    for t in range(8):
        n = int(rng.integers(1, 3000))
        sym = (rng.integers(0, 4, n) if t % 2 else np.tile(rng.integers(0, 4, 5), n)[:n]).astype(np.uint8)
        pats = [rng.integers(0, 4, int(rng.integers(0, 12))).astype(np.uint8) for _ in range(30)]
        for a in rng.integers(0, n, 30):
            p = sym[a:a + int(rng.integers(1, 41))].copy()
            if p.size > 3 and rng.random() < 0.4:
                p[int(rng.integers(0, p.size))] ^= 1
            pats.append(p)
        pats.append(np.concatenate([sym, sym[:9]]))
        cat, off, lens = oracle.pack_patterns(pats)
        got = oracle.scan_count_bucketed(sym, cat, off, lens)
        assert np.array_equal(got, oracle.scan_count(sym, cat, off, lens))
        if n <= 600:
            brute = [n + 1 if len(p) == 0 else sum(1 for i in range(n - len(p) + 1) if np.array_equal(sym[i:i + len(p)], p))
                     for p in pats]
            assert [int(x) for x in got] == brute
