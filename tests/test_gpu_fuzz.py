"""Randomised parity sweep: random sizes (incl. just below / above line and superblock
boundaries), random densities, every layout, random tuning knobs; bit-exact against the oracle."""
import numpy as np
import pytest

import gen
import oracle
import paper_2602_04103_b200 as qr
from _util import to_dev, to_host

pytestmark = pytest.mark.gpu

LAYOUTS = [qr.QR_LAYOUT_BIRANK16, qr.QR_LAYOUT_BIRANK64X2, qr.QR_LAYOUT_QUADRANK16, qr.QR_LAYOUT_QUADRANK64]
UNITS = {qr.QR_LAYOUT_BIRANK16: (496, 63488), qr.QR_LAYOUT_BIRANK64X2: (384, 192),
         qr.QR_LAYOUT_QUADRANK16: (224, 57344), qr.QR_LAYOUT_QUADRANK64: (128, 64)}


@pytest.mark.parametrize("trial", range(24))
def test_random_sizes_layouts_knobs(cuda, trial):
    import torch

    rng = np.random.default_rng(1000 + trial)
    layout = LAYOUTS[trial % 4]
    b, big = UNITS[layout]
    base = int(rng.choice([b, big, 1]))
    n = int(max(0, base * int(rng.integers(0, 40)) + int(rng.integers(-3, 4)))) if trial % 3 else int(rng.integers(0, 1 << 21))
    bits = layout in (qr.QR_LAYOUT_BIRANK16, qr.QR_LAYOUT_BIRANK64X2)
    if bits:
        p = float(rng.choice([0.5, 0.01, 0.99, 1.0]))
        w = gen.bits(int(rng.integers(1 << 30)), n, p)
    else:
        w = gen.dna(int(rng.integers(1 << 30)), n, int(n >= 2 * gen.BLOCK and trial % 2))
    m = int(rng.integers(1, 300000))
    q, c = gen.queries(int(rng.integers(1 << 30)), n, m, with_c=True)
    k = int(rng.choice([1, 2, 4, 8]))
    bps = int(rng.choice([1, 3, 16, 64]))
    qr.qr_set_tuning("rank_k", k)
    qr.qr_set_tuning("rank_blocks_per_sm", bps)
    qr.qr_set_tuning("rank_pair", int(rng.integers(0, 3)))
    try:
        h = qr.qr_build(w, n, layout)
        dq = to_dev(q, cuda)
        out = torch.empty_like(dq)
        if bits:
            qr.qr_rank(h, dq, None, out)
            torch.cuda.synchronize()
            ref = oracle.BitsOracle(w, n).rank(q)
            assert np.array_equal(to_host(out), ref)
        else:
            o4 = torch.empty((m, 4), dtype=torch.uint64, device=cuda)
            qr.qr_rank(h, dq, to_dev(c, cuda), out)
            qr.qr_rank_all4(h, dq, o4)
            torch.cuda.synchronize()
            ora = oracle.DnaOracle(w, n)
            assert np.array_equal(to_host(out), ora.rank(q, c))
            assert np.array_equal(to_host(o4), ora.rank_all4(q))
    finally:
        qr.qr_set_tuning("rank_k", 2)
        qr.qr_set_tuning("rank_blocks_per_sm", 64)
        qr.qr_set_tuning("rank_pair", 2)


@pytest.mark.parametrize("trial", range(8))
def test_random_fm(cuda, trial):
    import torch

    rng = np.random.default_rng(2000 + trial)
    n = int(rng.integers(1, 150000))
    w = gen.dna(int(rng.integers(1 << 30)), n, int(n >= 2 * gen.BLOCK and trial % 2))
    sym = gen.unpack_dna(w, n)
    fm = qr.qr_fm_build(w, n)
    pats = []
    for _ in range(1500):
        L = int(rng.integers(0, 60))
        if rng.random() < 0.5 and n > L:
            a = int(rng.integers(0, n - L + 1))
            p = sym[a:a + L].copy()
            if L and rng.random() < 0.3:
                j = int(rng.integers(0, L)); p[j] = (p[j] + 1) % 4
        else:
            p = rng.integers(0, 4, L).astype(np.uint8)
        pats.append(p)
    cat, off, lens = oracle.pack_patterns(pats)
    ref = oracle.scan_count(sym, cat, off, lens)
    qr.qr_set_tuning("fm_step", int(rng.integers(0, 4)))
    qr.qr_set_tuning("fm_blocks_per_sm", int(rng.choice([1, 4, 64])))
    try:
        d = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        qr.qr_fm_count(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, d, lens.size)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("fm_step", 0)
        qr.qr_set_tuning("fm_blocks_per_sm", 64)
    assert np.array_equal(to_host(d).view(np.uint32), ref)


@pytest.mark.parametrize("trial", range(6))
def test_random_fm_approx(cuda, trial):
    """Random text sizes / kinds, k-mer widths, BWT layouts, k in 0..3 and work orders: counts
    within Hamming distance k equal the oracle's direct scan."""
    import torch

    rng = np.random.default_rng(3000 + trial)
    n = int(rng.integers(1, 60000))
    w = gen.dna(int(rng.integers(1 << 30)), n, int(n >= 2 * gen.BLOCK and trial % 2))
    sym = gen.unpack_dna(w, n)
    kw = int(rng.choice([0, 4, 8, 10]))
    lay = [qr.QR_LAYOUT_QUADRANK16, qr.QR_LAYOUT_QUADRANK16X2][trial % 2]
    fm = qr.qr_fm_build(w, n, kmer_k=kw, bwt_layout=lay)
    k = trial % 4
    pats = []
    for _ in range(300 if k < 3 else 80):
        L = int(rng.integers(0, 30))
        if rng.random() < 0.5 and n > L:
            a = int(rng.integers(0, n - L + 1))
            p = sym[a:a + L].copy()
            for _s in range(int(rng.integers(0, 4))):
                if L:
                    j = int(rng.integers(0, L)); p[j] = (p[j] + 1 + rng.integers(0, 3)) % 4
        else:
            p = rng.integers(0, 4, L).astype(np.uint8)
        pats.append(p)
    cat, off, lens = oracle.pack_patterns(pats)
    ref = oracle.scan_count_hdk(sym, cat, off, lens, k)
    qr.qr_set_tuning("fm_dyn", int(rng.integers(0, 2)))
    try:
        d = torch.empty(lens.size, dtype=torch.int32, device=cuda)
        qr.qr_fm_count_approx(fm, to_dev(cat, cuda), to_dev(lens, cuda), 0, k, d, lens.size)
        torch.cuda.synchronize()
    finally:
        qr.qr_set_tuning("fm_dyn", 1)
    assert np.array_equal(to_host(d).view(np.uint32), ref)
