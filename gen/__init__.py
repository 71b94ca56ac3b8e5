"""Seeded, counter-based synthetic inputs (harness).

Serves both sides — the CPU oracle's tests and the CUDA product — and holds none
of the method's arithmetic (see ``gen/qrgen.h`` for the recipes).  Host fills are
plain C (``libqrgen_host.so``); device fills are CUDA kernels
(``libqrgen_dev.so``) producing bit-identical streams directly in HBM.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_H = None
_D = None
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)

BLOCK = 10000


def _host():
    global _H
    if _H is None:
        p = os.path.join(_HERE, "libqrgen_host.so")
        if not os.path.exists(p):
            raise RuntimeError(f"generator library missing: {p} (run `make`)")
        L = C.CDLL(p)
        L.qrgen_bits_host.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, u64p]
        L.qrgen_dna_host.argtypes = [C.c_uint64, C.c_uint64, C.c_int, u64p]
        L.qrgen_queries_host.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p, u8p]
        L.qrgen_patterns_host.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, u64p, C.c_uint64, u8p]
        L.qrgen_unpack_dna_host.argtypes = [u64p, C.c_uint64, u8p]
        L.qrgen_host_threads.restype = C.c_int
        for f in ("qrgen_bits_host", "qrgen_dna_host", "qrgen_queries_host", "qrgen_patterns_host", "qrgen_unpack_dna_host"):
            getattr(L, f).restype = None
        _H = L
    return _H


def _dev():
    global _D
    if _D is None:
        p = os.path.join(_HERE, "libqrgen_dev.so")
        if not os.path.exists(p):
            raise RuntimeError(f"generator library missing: {p} (run `make`)")
        L = C.CDLL(p)
        V = C.c_void_p
        L.qrgen_bits_dev.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, V, V]
        L.qrgen_dna_dev.argtypes = [C.c_uint64, C.c_uint64, C.c_int, V, V]
        L.qrgen_queries_dev.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, V, V, V]
        L.qrgen_patterns_dev.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, V, C.c_uint64, V, V]
        for f in ("qrgen_bits_dev", "qrgen_dna_dev", "qrgen_queries_dev", "qrgen_patterns_dev"):
            getattr(L, f).restype = C.c_int
        _D = L
    return _D


def p_threshold(p: float) -> tuple[int, int]:
    """(word_mode, thr): p = 0.5 uses whole random words; otherwise bit i = [h < p*2^64]."""
    if p == 0.5:
        return 1, 0
    if p >= 1.0:
        return 0, (1 << 64) - 1
    return 0, int(p * 2.0**64)


def _ptr(a):
    return a.ctypes.data_as(u64p)


# ------------------------------------------------------------------ host
def bits(seed: int, n: int, p: float = 0.5) -> np.ndarray:
    wm, thr = p_threshold(p)
    out = np.empty(max(1, (n + 63) >> 6), dtype=np.uint64)
    out[-1] = 0
    _host().qrgen_bits_host(seed, n, wm, thr, _ptr(out))
    return out


def dna(seed: int, n: int, kind: int = 0) -> np.ndarray:
    """kind 0 = iid uniform ACGT; kind 1 = block-repeat (config 5)."""
    out = np.empty(max(1, (n + 31) >> 5), dtype=np.uint64)
    out[-1] = 0
    _host().qrgen_dna_host(seed, n, kind, _ptr(out))
    return out


def queries(seed: int, n: int, m: int, i0: int = 0, with_c: bool = False):
    q = np.empty(m, dtype=np.uint64)
    c = np.empty(m, dtype=np.uint8) if with_c else None
    _host().qrgen_queries_host(seed, n, i0, m, _ptr(q), c.ctypes.data_as(u8p) if with_c else None)
    return (q, c) if with_c else q


def patterns(seed: int, kind: int, m: int, length: int, text2b: np.ndarray, n: int, i0: int = 0) -> np.ndarray:
    out = np.empty(max(1, m * length), dtype=np.uint8)
    _host().qrgen_patterns_host(seed, kind, i0, m, length, _ptr(text2b), n, out.ctypes.data_as(u8p))
    return out[: m * length]


def unpack_dna(words: np.ndarray, n: int) -> np.ndarray:
    out = np.empty(max(1, n), dtype=np.uint8)
    _host().qrgen_unpack_dna_host(_ptr(words), n, out.ctypes.data_as(u8p))
    return out[:n]


def host_threads() -> int:
    return int(_host().qrgen_host_threads())


# ------------------------------------------------------------------ device (torch tensors)
def _stream(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _chk(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: cuda error {rc}")


def bits_dev(seed: int, n: int, p: float, out, stream=None):
    wm, thr = p_threshold(p)
    _chk(_dev().qrgen_bits_dev(seed, n, wm, thr, C.c_void_p(out.data_ptr()), _stream(stream)), "qrgen_bits_dev")


def dna_dev(seed: int, n: int, kind: int, out, stream=None):
    _chk(_dev().qrgen_dna_dev(seed, n, kind, C.c_void_p(out.data_ptr()), _stream(stream)), "qrgen_dna_dev")


def queries_dev(seed: int, n: int, m: int, q, c=None, i0: int = 0, stream=None):
    _chk(_dev().qrgen_queries_dev(seed, n, i0, m, C.c_void_p(q.data_ptr()) if q is not None else None,
                                  C.c_void_p(c.data_ptr()) if c is not None else None, _stream(stream)), "qrgen_queries_dev")


def patterns_dev(seed: int, kind: int, m: int, length: int, text2b, n: int, out, i0: int = 0, stream=None):
    _chk(_dev().qrgen_patterns_dev(seed, kind, i0, m, length, C.c_void_p(text2b.data_ptr()), n,
                                   C.c_void_p(out.data_ptr()), _stream(stream)), "qrgen_patterns_dev")
