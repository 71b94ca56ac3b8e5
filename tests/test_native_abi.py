"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/qrank.h
declares, and validates arguments (status codes, error strings) before touching a GPU."""
import ctypes as C
import os
import re

import pytest

import paper_2602_04103_b200 as qr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "qrank.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qr_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("qr_birank_build", "qr_quadrank_build", "qr_rank", "qr_rank_all4", "qr_fm_build", "qr_fm_count",
                 "qr_free", "qr_fm_free", "qr_last_error"):
        assert must in syms
    assert set(syms) == set(qr.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = C.CDLL(qr.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(L, s), s


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", qr.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_product_does_not_reference_oracle():
    pkg = os.path.join(ROOT, "paper_2602_04103_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in txt.replace("no oracle", ""), f


def test_argument_validation_without_gpu():
    L = qr.lib()
    assert L.qr_rank(None, None, None, None, 5, None) == qr.QR_EINVAL
    assert b"null handle" in L.qr_last_error()
    assert L.qr_rank(None, None, None, None, 0, None) == qr.QR_EINVAL      # null handle still invalid
    out = C.c_void_p()
    assert L.qr_birank_build(C.c_void_p(8), 1 << 43, 0, None, C.byref(out)) == qr.QR_ECAPACITY
    assert b"2^43" in L.qr_last_error()
    assert L.qr_quadrank_build(C.c_void_p(8), 1 << 45, 0, None, C.byref(out)) == qr.QR_ECAPACITY
    assert L.qr_fm_build(C.c_void_p(8), (1 << 32) - 1, None, 0, None, C.byref(out)) == qr.QR_ECAPACITY
    assert L.qr_fm_build(C.c_void_p(8), 0, None, 0, None, C.byref(out)) == qr.QR_EINVAL
    assert L.qr_birank_build(None, 10, 0, None, C.byref(out)) == qr.QR_EINVAL
    assert L.qr_set_tuning(b"rank_k", 3) == qr.QR_EINVAL
    assert L.qr_set_tuning(b"nope", 1) == qr.QR_EINVAL
    assert L.qr_set_tuning(b"rank_k", 4) == qr.QR_OK
    L.qr_free(None)
    L.qr_fm_free(None)
    with pytest.raises(qr.QrError):
        qr.qr_set_tuning("rank_blocks_per_sm", 0)


def test_binding_rejects_wrong_dtypes():
    """The binding refuses arrays too small for the call (e.g. an int32 query array)."""
    import numpy as np

    h = object.__new__(qr.Index)          # never reaches the library: the size check fires first
    with pytest.raises(qr.QrError):
        qr.qr_rank(h, np.zeros(10, np.int32), None, np.zeros(10, np.uint64))
    with pytest.raises(qr.QrError):
        qr.qr_rank(h, np.zeros(10, np.uint64), None, np.zeros(5, np.uint64))
    with pytest.raises(qr.QrError):
        qr.qr_rank_all4(h, np.zeros(10, np.uint64), np.zeros(10, np.uint64))
