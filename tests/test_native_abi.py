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
    assert L.qr_build(C.c_void_p(8), 1 << 40, qr.QR_LAYOUT_BIRANK16X2, 0, None, C.byref(out)) == qr.QR_ECAPACITY
    assert L.qr_build(C.c_void_p(8), 1 << 39, qr.QR_LAYOUT_QUADRANK16X2, 0, None, C.byref(out)) == qr.QR_ECAPACITY
    assert L.qr_build(C.c_void_p(8), 10, 99, 0, None, C.byref(out)) == qr.QR_EINVAL         # unknown layout
    assert b"bad layout" in L.qr_last_error()
    assert L.qr_fm_build_opts(C.c_void_p(8), 10, None, 8, qr.QR_LAYOUT_BIRANK16, 0, None, C.byref(out)) == qr.QR_EINVAL
    assert L.qr_fm_build_opts(C.c_void_p(8), 10, None, 15, qr.QR_LAYOUT_QUADRANK16, 0, None, C.byref(out)) == qr.QR_EINVAL
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
    with pytest.raises(qr.QrError):
        qr.qr_rank_chain(h, np.zeros(10, np.uint64), None, np.zeros(10, np.uint32), 5)
    with pytest.raises(qr.QrError):
        qr.qr_gather_ceiling(h, np.zeros(10, np.uint64), np.zeros(9, np.uint64))
    fm = object.__new__(qr.Fm)
    pats = np.zeros(10 * 32, np.uint8)
    with pytest.raises(qr.QrError):      # patterns too short for m * fixed_len
        qr.qr_fm_count(fm, pats[:-1], None, 32, np.zeros(10, np.uint32), 10)
    with pytest.raises(qr.QrError):      # reverse-complement output too short
        qr.qr_fm_count_both(fm, pats, None, 32, np.zeros(10, np.uint32), np.zeros(9, np.uint32), 10)
    with pytest.raises(qr.QrError):      # u64 counts where the ABI writes u32
        qr.qr_fm_count_approx(fm, pats, None, 32, 1, np.zeros(10, np.uint64), 10)
    with pytest.raises(qr.QrError):      # lengths must be u32
        qr.qr_fm_count_work(fm, pats, np.full(10, 32, np.int64), 0, np.zeros(10, np.uint32), 10,
                            np.zeros(2, np.uint64))


def test_binding_rejects_strided_and_short_buffers():
    """Strided views (numpy slices, negative strides, torch transposes and stride-0 expansions) and
    build inputs shorter than n symbols are refused before any pointer reaches the library."""
    import numpy as np
    import torch

    h = object.__new__(qr.Index)
    q = np.zeros(20, np.uint64)
    with pytest.raises(qr.QrError, match="contiguous"):
        qr.qr_rank(h, q[::2], None, np.zeros(10, np.uint64))
    with pytest.raises(qr.QrError, match="contiguous"):
        qr.qr_rank(h, q[:10], None, np.zeros(20, np.uint64)[::-2])
    with pytest.raises(qr.QrError, match="contiguous"):
        qr.qr_rank_all4(h, torch.zeros(10, dtype=torch.uint64), torch.zeros(4, 10, dtype=torch.uint64).t())
    with pytest.raises(qr.QrError, match="zero stride|contiguous"):
        qr.qr_rank(h, torch.zeros(1, dtype=torch.uint64).expand(10), None, torch.zeros(10, dtype=torch.uint64))
    fm = object.__new__(qr.Fm)
    with pytest.raises(qr.QrError, match="contiguous"):   # variable-length patterns, strided
        qr.qr_fm_count(fm, np.zeros(64, np.uint8)[::2], np.full(2, 16, np.uint32), 0, np.zeros(2, np.uint32), 2)
    with pytest.raises(qr.QrError):                        # 2^12 bits need 64 words
        qr.qr_birank_build(np.zeros(63, np.uint64), 1 << 12)
    with pytest.raises(qr.QrError):                        # 1000 chars need 32 words
        qr.qr_quadrank_build(np.zeros(31, np.uint64), 1000)
    with pytest.raises(qr.QrError):
        qr.qr_build(np.zeros(31, np.uint64), 1000, qr.QR_LAYOUT_QUADRANK64)
    with pytest.raises(qr.QrError):                        # SA of n + 1 rows
        qr.qr_fm_build(np.zeros(32, np.uint64), 1000, sa=np.zeros(1000, np.uint32))
    with pytest.raises(qr.QrError, match="contiguous"):
        qr.qr_import_layout(np.zeros(256, np.uint8)[::2], None, 10, qr.QR_LAYOUT_BIRANK64X2)


def test_device_index_normalisation():
    import torch

    from paper_2602_04103_b200.multigpu import device_index

    assert device_index(3) == 3
    assert device_index("cuda:2") == 2
    assert device_index(torch.device("cuda", 5)) == 5
    with pytest.raises(ValueError):
        device_index("cpu")


def test_tuning_knob_validation():
    """Every launch knob accepts its documented values and rejects the rest (QR_EINVAL, message
    set); the (K, CTA threads) pairs of the cluster kernels are checked against the instantiated
    set.  Defaults are restored afterwards (knobs are process-wide)."""
    L = qr.lib()
    ok = {
        "rank_smem": [0, 1, 2], "rank_dyn": [0, 1], "rank_smem_k": [0, 1, 2, 3, 4, 6, 8],
        "rank_smem_clusters": [0, 1, 74, 4096], "fm_dyn": [0, 1], "fm_seed": [0, 1, 2], "fm_smem": [0, 1, 2],
        "fm_step": [0, 1, 2, 3, 4], "fm_packed": [0, 1], "fm_kbits": [0, 1, 2], "check_range": [0, 1], "fm_refill": [0, 1, 8, 32], "rank_pair": [0, 1, 2], "rank_s_lane": [0, 1], "index64": [0, 1],
        "rank_k": [1, 2, 4, 8], "rank_blocks_per_sm": [1, 64], "fm_blocks_per_sm": [1, 64],
        "stage_slots": [2, 4], "stage_chunk": [1024, 1 << 23], "rank_resident": [0, 1], "rank_big_pack": [0, 1],
        "rank_big_cs": [0, 4, 8, 16],
    }
    bad = {
        "rank_smem": [-1, 3], "rank_dyn": [2], "rank_smem_k": [5, 7, 16], "rank_smem_clusters": [-1, 4097],
        "fm_dyn": [2], "fm_seed": [3], "fm_smem": [3], "fm_step": [5, -1], "fm_packed": [2], "fm_kbits": [3, -1], "check_range": [2, -1], "fm_refill": [-1, 33], "rank_pair": [3, -1], "rank_s_lane": [2],
        "index64": [2], "rank_k": [0, 3], "rank_blocks_per_sm": [0, 65], "fm_blocks_per_sm": [0, 65],
        "stage_slots": [1, 5], "stage_chunk": [1023], "rank_resident": [2, -1], "rank_big_pack": [2],
        "rank_big_cs": [2, 32],
    }
    try:
        for key, vals in ok.items():
            for v in vals:
                assert L.qr_set_tuning(key.encode(), v) == qr.QR_OK, (key, v)
        for key, vals in bad.items():
            for v in vals:
                assert L.qr_set_tuning(key.encode(), v) == qr.QR_EINVAL, (key, v)
                assert key.encode() in L.qr_last_error() or b"must" in L.qr_last_error(), (key, L.qr_last_error())
        # (K, threads) pairs: 4 @ 768 and 6 @ 768 and 8 @ 512 exist; 2 @ 768 and 8 @ 1024 do not
        for k, t, st in ((4, 768, qr.QR_OK), (6, 768, qr.QR_OK), (8, 512, qr.QR_OK), (2, 768, qr.QR_EINVAL),
                         (8, 1024, qr.QR_EINVAL), (3, 1024, qr.QR_OK)):
            assert L.qr_set_tuning(b"rank_smem_k", k) == qr.QR_OK
            assert L.qr_set_tuning(b"rank_smem_threads", t) == st, (k, t)
    finally:
        for key, v in (("rank_smem", 1), ("rank_dyn", 1), ("rank_smem_k", 0), ("rank_smem_clusters", 0), ("fm_dyn", 1),
                       ("fm_seed", 0), ("fm_smem", 1), ("fm_step", 0), ("fm_packed", 1), ("fm_kbits", 0), ("check_range", 0), ("fm_refill", 0), ("rank_pair", 2), ("rank_s_lane", 1),
                       ("index64", 0), ("rank_k", 2), ("rank_blocks_per_sm", 64), ("fm_blocks_per_sm", 64),
                       ("stage_slots", 3), ("stage_chunk", 1 << 23), ("rank_resident", 1), ("rank_big_pack", 0),
                       ("rank_big_cs", 0)):
            L.qr_set_tuning(key.encode(), v)


@pytest.mark.parametrize("compiler,std", [("gcc", "-std=c99"), ("g++", "-std=c++17")])
def test_header_compiles_and_links_from_plain_c(tmp_path, compiler, std):
    """include/qrank.h is self-contained C (and C++): a translation unit taking the address of
    every declared function compiles warning-free and links against libqrank.so alone."""
    import subprocess

    syms = declared_symbols()
    src = '#include "qrank.h"\n#include <stdio.h>\nint main(void) {\n  const void* fns[] = {\n'
    src += ",\n".join(f"    (const void*)&{s}" for s in syms) + "\n  };\n"
    src += '  printf("%d\\n", (int)(sizeof(fns) / sizeof(fns[0])));\n  return 0;\n}\n'
    f = tmp_path / ("t.c" if compiler == "gcc" else "t.cpp")
    f.write_text(src)
    exe = tmp_path / "t"
    libdir = os.path.dirname(qr.LIB_PATH)
    r = subprocess.run([compiler, std, "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), str(f),
                        "-o", str(exe), "-L", libdir, "-lqrank", f"-Wl,-rpath,{libdir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and int(out.stdout.strip()) == len(syms)


def test_c_demo_is_built():
    assert os.access(os.path.join(ROOT, "examples", "qrank_demo"), os.X_OK)


@pytest.mark.gpu
def test_c_demo_runs(cuda):
    """examples/qrank_demo.c: BiRank / QuadRank / QuadFm from plain C with host buffers,
    checked against naive loops inside the program."""
    import subprocess

    r = subprocess.run([os.path.join(ROOT, "examples", "qrank_demo")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "qrank_demo OK" in r.stdout
