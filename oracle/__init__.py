"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product package
``paper_2602_04103_b200`` never imports it, and the two share no code (see
``oracle/oracle.c`` for the definitions it computes and the paper passages they
follow: rank = PAPER.md:61-63, FM backward search = PAPER.md:922-928).

Thin ctypes marshalling over ``oracle/liboracle.so`` (plain C, built by the root
``Makefile``); numpy arrays in, numpy arrays out.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u8p = C.POINTER(C.c_uint8)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library missing: {path} (run `make` at the repo root)")
        L = C.CDLL(path)
        sig = {
            "or_bits_prefix": [u64p, C.c_uint64, u64p],
            "or_rank_bits": [u64p, u64p, C.c_uint64, u64p, u8p, C.c_uint64, u64p],
            "or_dna_checkpoints": [u64p, C.c_uint64, u64p],
            "or_rank_dna": [u64p, u64p, C.c_uint64, u64p, u8p, C.c_uint64, u64p],
            "or_rank_all4_dna": [u64p, u64p, C.c_uint64, u64p, C.c_uint64, u64p],
            "or_suffix_array": [u8p, C.c_uint64, u32p],
            "or_bwt": [u8p, C.c_uint64, u32p, u8p, u64p],
            "or_fm_prepare": [u8p, C.c_uint64, u64p, u64p],
            "or_fm_count": [u8p, u64p, u64p, C.c_uint64, u8p, u64p, u32p, C.c_uint64, u32p, u32p],
            "or_fm_work": [u8p, u64p, u64p, C.c_uint64, u8p, u64p, u32p, C.c_uint64, C.c_uint32, C.c_uint64, u64p, u64p],
            "or_sa_count": [u8p, C.c_uint64, u32p, u8p, u64p, u32p, C.c_uint64, u32p],
            "or_scan_count": [u8p, C.c_uint64, u8p, u64p, u32p, C.c_uint64, u32p],
            "or_scan_count_bucketed": [u8p, C.c_uint64, u8p, u64p, u32p, C.c_uint64, u32p],
            "or_scan_count_hd1": [u8p, C.c_uint64, u8p, u64p, u32p, C.c_uint64, u32p],
            "or_scan_count_hdk": [u8p, C.c_uint64, u8p, u64p, u32p, C.c_uint64, C.c_uint32, u32p],
            "or_threads": [],
            "or_set_threads": [C.c_int],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int if name in ("or_suffix_array", "or_threads") else None
        _LIB = L
    return _LIB


def _p(a, t):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


def threads() -> int:
    return int(lib().or_threads())


def set_threads(n: int) -> None:
    """Parallel-for width of the oracle (all host cores for the timed CPU baseline)."""
    lib().or_set_threads(int(n))


# ------------------------------------------------------------------ sigma = 2
class BitsOracle:
    """rank(q) = sum_{i<q} t_i over LE-packed bits."""

    def __init__(self, words: np.ndarray, n: int):
        self.words = np.ascontiguousarray(words, dtype=np.uint64)
        self.n = int(n)
        self.W = np.empty(self.words.size + 1, dtype=np.uint64)
        lib().or_bits_prefix(_p(self.words, u64p), self.words.size, _p(self.W, u64p))

    def rank(self, q: np.ndarray, c: np.ndarray | None = None) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.uint64)
        out = np.empty(q.size, dtype=np.uint64)
        if c is not None:
            c = np.ascontiguousarray(c, dtype=np.uint8)
        lib().or_rank_bits(_p(self.words, u64p), _p(self.W, u64p), self.n, _p(q, u64p), _p(c, u8p), q.size, _p(out, u64p))
        return out


# ------------------------------------------------------------------ sigma = 4
class DnaOracle:
    """rank(q, c) = sum_{i<q} [t_i = c] over 2-bit LE-packed DNA."""

    def __init__(self, words: np.ndarray, n: int):
        self.words = np.ascontiguousarray(words, dtype=np.uint64)
        self.n = int(n)
        nw = (self.n + 31) >> 5
        self.cp = np.empty(4 * (nw + 1), dtype=np.uint64)
        lib().or_dna_checkpoints(_p(self.words, u64p), self.n, _p(self.cp, u64p))

    def rank(self, q: np.ndarray, c: np.ndarray) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.uint64)
        c = np.ascontiguousarray(c, dtype=np.uint8)
        out = np.empty(q.size, dtype=np.uint64)
        lib().or_rank_dna(_p(self.words, u64p), _p(self.cp, u64p), self.n, _p(q, u64p), _p(c, u8p), q.size, _p(out, u64p))
        return out

    def rank_all4(self, q: np.ndarray) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.uint64)
        out = np.empty(4 * q.size, dtype=np.uint64)
        lib().or_rank_all4_dna(_p(self.words, u64p), _p(self.cp, u64p), self.n, _p(q, u64p), q.size, _p(out, u64p))
        return out.reshape(-1, 4)


# ------------------------------------------------------------------ FM
def suffix_array(sym: np.ndarray) -> np.ndarray:
    """SA of sym + '$' (n+1 entries), plain prefix doubling."""
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    sa = np.empty(sym.size + 1, dtype=np.uint32)
    if lib().or_suffix_array(_p(sym, u8p), sym.size, _p(sa, u32p)) != 0:
        raise MemoryError("or_suffix_array")
    return sa


def pack_patterns(patterns):
    """list of 1-D uint8 arrays -> (concat, offsets u64, lengths u32)."""
    lens = np.array([len(p) for p in patterns], dtype=np.uint32)
    off = np.zeros(len(patterns), dtype=np.uint64)
    if len(patterns) > 1:
        off[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
    cat = np.concatenate([np.asarray(p, dtype=np.uint8) for p in patterns]) if len(patterns) else np.zeros(0, np.uint8)
    if cat.size == 0:
        cat = np.zeros(1, dtype=np.uint8)
    return np.ascontiguousarray(cat), off, lens


class FmOracle:
    """Count-only FM index over a plain BWT with '$' = 4."""

    def __init__(self, sym: np.ndarray, sa: np.ndarray | None = None):
        self.sym = np.ascontiguousarray(sym, dtype=np.uint8)
        self.n = int(self.sym.size)
        self.sa = suffix_array(self.sym) if sa is None else np.ascontiguousarray(sa, dtype=np.uint32)
        self.bwt = np.empty(self.n + 1, dtype=np.uint8)
        sp = C.c_uint64(0)
        lib().or_bwt(_p(self.sym, u8p), self.n, _p(self.sa, u32p), _p(self.bwt, u8p), C.byref(sp))
        self.spos = int(sp.value)
        self.C = np.empty(5, dtype=np.uint64)
        self.cp = np.empty(5 * ((self.n + 1) // 64 + 1), dtype=np.uint64)
        lib().or_fm_prepare(_p(self.bwt, u8p), self.n + 1, _p(self.C, u64p), _p(self.cp, u64p))

    def _pk(self, cat, off, lens):
        return (np.ascontiguousarray(cat, dtype=np.uint8), np.ascontiguousarray(off, dtype=np.uint64),
                np.ascontiguousarray(lens, dtype=np.uint32))

    def count(self, cat, off, lens, with_steps=False):
        cat, off, lens = self._pk(cat, off, lens)
        out = np.empty(lens.size, dtype=np.uint32)
        steps = np.empty(lens.size, dtype=np.uint32) if with_steps else None
        lib().or_fm_count(_p(self.bwt, u8p), _p(self.cp, u64p), _p(self.C, u64p), self.n + 1,
                          _p(cat, u8p), _p(off, u64p), _p(lens, u32p), lens.size, _p(out, u32p), _p(steps, u32p))
        return (out, steps) if with_steps else out

    def work(self, cat, off, lens, skip=8, block=224):
        cat, off, lens = self._pk(cat, off, lens)
        ts, tl = C.c_uint64(0), C.c_uint64(0)
        lib().or_fm_work(_p(self.bwt, u8p), _p(self.cp, u64p), _p(self.C, u64p), self.n + 1,
                         _p(cat, u8p), _p(off, u64p), _p(lens, u32p), lens.size, skip, block, C.byref(ts), C.byref(tl))
        return int(ts.value), int(tl.value)

    def sa_count(self, cat, off, lens):
        cat, off, lens = self._pk(cat, off, lens)
        out = np.empty(lens.size, dtype=np.uint32)
        lib().or_sa_count(_p(self.sym, u8p), self.n, _p(self.sa, u32p), _p(cat, u8p), _p(off, u64p),
                          _p(lens, u32p), lens.size, _p(out, u32p))
        return out


def scan_count(sym: np.ndarray, cat, off, lens) -> np.ndarray:
    """Occurrences of each pattern by a direct scan of every text position."""
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    cat = np.ascontiguousarray(cat, dtype=np.uint8)
    off = np.ascontiguousarray(off, dtype=np.uint64)
    lens = np.ascontiguousarray(lens, dtype=np.uint32)
    out = np.empty(lens.size, dtype=np.uint32)
    lib().or_scan_count(_p(sym, u8p), sym.size, _p(cat, u8p), _p(off, u64p), _p(lens, u32p), lens.size, _p(out, u32p))
    return out


def scan_count_bucketed(sym: np.ndarray, cat, off, lens) -> np.ndarray:
    """Occurrences by a direct scan of every text position, patterns of >= 8 symbols grouped by
    their first 8 (the same counts as scan_count; for large batches on large texts)."""
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    cat = np.ascontiguousarray(cat, dtype=np.uint8)
    off = np.ascontiguousarray(off, dtype=np.uint64)
    lens = np.ascontiguousarray(lens, dtype=np.uint32)
    out = np.empty(lens.size, dtype=np.uint32)
    lib().or_scan_count_bucketed(_p(sym, u8p), sym.size, _p(cat, u8p), _p(off, u64p), _p(lens, u32p), lens.size,
                                 _p(out, u32p))
    return out


def scan_count_hd1(sym: np.ndarray, cat, off, lens) -> np.ndarray:
    """Positions where each pattern matches with at most one substitution (direct scan)."""
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    cat = np.ascontiguousarray(cat, dtype=np.uint8)
    off = np.ascontiguousarray(off, dtype=np.uint64)
    lens = np.ascontiguousarray(lens, dtype=np.uint32)
    out = np.empty(lens.size, dtype=np.uint32)
    lib().or_scan_count_hd1(_p(sym, u8p), sym.size, _p(cat, u8p), _p(off, u64p), _p(lens, u32p), lens.size,
                            _p(out, u32p))
    return out


def scan_count_hdk(sym: np.ndarray, cat, off, lens, k: int) -> np.ndarray:
    """Positions where each pattern matches with at most k substitutions (direct scan)."""
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    cat = np.ascontiguousarray(cat, dtype=np.uint8)
    off = np.ascontiguousarray(off, dtype=np.uint64)
    lens = np.ascontiguousarray(lens, dtype=np.uint32)
    out = np.empty(lens.size, dtype=np.uint32)
    lib().or_scan_count_hdk(_p(sym, u8p), sym.size, _p(cat, u8p), _p(off, u64p), _p(lens, u32p), lens.size, int(k),
                            _p(out, u32p))
    return out
