"""B200-native BiRank / QuadRank / QuadFm (arXiv 2602.04103) — Python binding.

Thin ctypes marshalling over the C-ABI library ``lib/libqrank.so`` (declared in
``include/qrank.h``).  Every function here has the C name and only turns
arguments into pointers/sizes: every step of the method runs in the library's
CUDA kernels.  There is no fallback — if the library is missing, importing the
binding raises.

Arrays may be torch tensors (device tensors on the handle's device, or CPU
tensors) or numpy arrays (host).  All query arrays of one call must live in the
same space (all device = one asynchronous kernel launch on ``stream``; all host =
the library's staged, pipelined host<->device path).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libqrank.so")

QR_OK, QR_EINVAL, QR_ECAPACITY, QR_ENOMEM, QR_ECUDA, QR_ERANGE = 0, 1, 2, 3, 4, 5
QR_LAYOUT_BIRANK16, QR_LAYOUT_BIRANK64X2, QR_LAYOUT_QUADRANK16, QR_LAYOUT_QUADRANK64, QR_LAYOUT_BIRANK16X2 = 1, 2, 3, 4, 5
QR_LAYOUT_QUADRANK16X2, QR_LAYOUT_BIRANK32X2 = 6, 7
_STATUS = {1: "QR_EINVAL", 2: "QR_ECAPACITY", 3: "QR_ENOMEM", 4: "QR_ECUDA", 5: "QR_ERANGE"}

# every symbol include/qrank.h declares (tests check the .so exports all of them)
EXPORTS = (
    "qr_birank_build", "qr_quadrank_build", "qr_rank", "qr_rank_all4", "qr_fm_build", "qr_fm_count", "qr_fm_count_both", "qr_fm_count_approx",
    "qr_fm_count_work", "qr_gather_ceiling", "qr_info", "qr_export_layout", "qr_fm_info", "qr_fm_export_kmer",
    "qr_clone_to_device", "qr_fm_clone_to_device", "qr_sync", "qr_free", "qr_fm_free", "qr_last_error",
    "qr_version", "qr_set_tuning", "qr_build", "qr_layout", "qr_rank_chain", "qr_import_layout", "qr_fm_build_ex", "qr_fm_kmer_width",
    "qr_super_cache_bytes", "qr_super_cache_clusters", "qr_fm_build_opts", "qr_fm_count_approx_both",
    "qr_fm_count_work_ex", "qr_checksum", "qr_fm_build_u8",
)


class QrError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libqrank.so (raises if it was not built — no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libqrank.so not built: {LIB_PATH} (run `make` at the repo root)")
        L = C.CDLL(LIB_PATH)
        V, U64, I32, U32 = C.c_void_p, C.c_uint64, C.c_int, C.c_uint32
        PP = C.POINTER(C.c_void_p)
        sig = {
            "qr_birank_build": ([V, U64, I32, V, PP], I32),
            "qr_quadrank_build": ([V, U64, I32, V, PP], I32),
            "qr_rank": ([V, V, V, V, U64, V], I32),
            "qr_rank_all4": ([V, V, V, U64, V], I32),
            "qr_fm_build": ([V, U64, V, I32, V, PP], I32),
            "qr_fm_count": ([V, V, V, U32, V, U64, V], I32),
            "qr_fm_count_work": ([V, V, V, U32, V, U64, V, V], I32),
            "qr_fm_count_both": ([V, V, V, U32, V, V, U64, V], I32),
            "qr_fm_count_work_ex": ([V, V, V, U32, U32, V, V, U64, V, V], I32),
            "qr_checksum": ([V, U64, C.c_int, U64, V, V], I32),
            "qr_fm_build_u8": ([V, U64, V, I32, V, PP], I32),
            "qr_fm_count_approx": ([V, V, V, U32, U32, V, U64, V], I32),
            "qr_fm_count_approx_both": ([V, V, V, U32, U32, V, V, U64, V], I32),
            "qr_gather_ceiling": ([V, V, V, U64, I32, V], I32),
            "qr_info": ([V, C.POINTER(U64), C.POINTER(C.c_int), C.POINTER(U64), C.POINTER(U64)], I32),
            "qr_export_layout": ([V, V, V], I32),
            "qr_fm_info": ([V, C.POINTER(U64), C.POINTER(U64), C.POINTER(U64), PP], I32),
            "qr_fm_export_kmer": ([V, V], I32),
            "qr_clone_to_device": ([V, I32, V, PP], I32),
            "qr_fm_clone_to_device": ([V, I32, V, PP], I32),
            "qr_sync": ([V], I32),
            "qr_free": ([V], None),
            "qr_fm_free": ([V], None),
            "qr_last_error": ([], C.c_char_p),
            "qr_version": ([], C.c_char_p),
            "qr_set_tuning": ([C.c_char_p, C.c_int64], I32),
            "qr_build": ([V, U64, I32, I32, V, PP], I32),
            "qr_layout": ([V, C.POINTER(C.c_int)], I32),
            "qr_rank_chain": ([V, V, V, V, U64, U64, V], I32),
            "qr_import_layout": ([V, U64, V, U64, U64, I32, I32, V, PP], I32),
            "qr_fm_build_ex": ([V, U64, V, I32, I32, V, PP], I32),
            "qr_fm_kmer_width": ([V, C.POINTER(C.c_int)], I32),
            "qr_fm_build_opts": ([V, U64, V, I32, I32, I32, V, PP], I32),
            "qr_super_cache_bytes": ([V, C.POINTER(U64)], I32),
            "qr_super_cache_clusters": ([V, C.POINTER(C.c_int)], I32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(st: int, where: str):
    if st != QR_OK:
        raise QrError(st, where, lib().qr_last_error().decode())


def _ptr(a):
    """data pointer of a torch tensor / numpy array / int / None."""
    if a is None:
        return None
    if isinstance(a, int):
        return C.c_void_p(a)
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    if hasattr(a, "ctypes"):
        return C.c_void_p(a.ctypes.data)
    raise TypeError(f"cannot take a pointer of {type(a)}")


def _nbytes_item(a):
    """(element size, element count) of a torch tensor / numpy array, or None for raw pointers."""
    if a is None or isinstance(a, int):
        return None
    if hasattr(a, "element_size"):
        return a.element_size(), a.numel()
    if hasattr(a, "itemsize"):
        return a.itemsize, a.size
    return None


def _contig(a, name: str):
    """Reject strided views (torch non-contiguous, stride-0 expansions; numpy non-C-contiguous or
    negative strides): the library reads and writes dense arrays from the data pointer."""
    if a is None or isinstance(a, int):
        return
    if hasattr(a, "is_contiguous"):
        if not a.is_contiguous():
            raise QrError(QR_EINVAL, name, "tensor is not contiguous")
        if a.numel() > 1 and any(st == 0 for st, sz in zip(a.stride(), a.shape) if sz > 1):
            raise QrError(QR_EINVAL, name, "tensor has a zero stride")
    elif hasattr(a, "flags"):
        if not a.flags["C_CONTIGUOUS"] or any(st < 0 for st in a.strides):
            raise QrError(QR_EINVAL, name, "array is not C-contiguous")


def _need(a, itemsize: int, count: int, name: str):
    """Reject arrays whose element size or length cannot hold `count` items, or that are not
    dense (marshalling check: a wrong dtype or a strided view would otherwise be read or written
    out of bounds by the kernels)."""
    info = _nbytes_item(a)
    if info is None:
        return
    _contig(a, name)
    es, n = info
    if es * n < itemsize * count or (es != itemsize and itemsize in (1, 4, 8) and es not in (itemsize,)):
        raise QrError(QR_EINVAL, name, f"needs {count} items of {itemsize} B, got {n} of {es} B")


def _stream(s):
    if s is None:
        try:
            import torch

            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return None
    if isinstance(s, int):
        return C.c_void_p(s)
    return C.c_void_p(s.cuda_stream)


class Index:
    """Owning wrapper of a qr_index* (BiRank16 or QuadRank16)."""

    def __init__(self, ptr: int, owned: bool = True):
        self.ptr = C.c_void_p(ptr)
        self.owned = owned
        n, sig, lb, sb = C.c_uint64(), C.c_int(), C.c_uint64(), C.c_uint64()
        _check(lib().qr_info(self.ptr, C.byref(n), C.byref(sig), C.byref(lb), C.byref(sb)), "qr_info")
        self.n, self.sigma, self.line_bytes, self.super_bytes = n.value, sig.value, lb.value, sb.value
        lay = C.c_int()
        _check(lib().qr_layout(self.ptr, C.byref(lay)), "qr_layout")
        self.layout = lay.value

    def free(self):
        if self.owned and self.ptr:
            lib().qr_free(self.ptr)
        self.ptr = C.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Fm:
    """Owning wrapper of a qr_fm*."""

    def __init__(self, ptr: int):
        self.ptr = C.c_void_p(ptr)
        n, sp = C.c_uint64(), C.c_uint64()
        Cs = (C.c_uint64 * 5)()
        bw = C.c_void_p()
        _check(lib().qr_fm_info(self.ptr, C.byref(n), C.byref(sp), Cs, C.byref(bw)), "qr_fm_info")
        self.n, self.spos, self.C = n.value, sp.value, list(Cs)
        self.bwt = Index(bw.value, owned=False)
        kk = C.c_int()
        _check(lib().qr_fm_kmer_width(self.ptr, C.byref(kk)), "qr_fm_kmer_width")
        self.kmer_k = kk.value

    def free(self):
        if self.ptr:
            lib().qr_fm_free(self.ptr)
        self.ptr = C.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ----------------------------------------------------------------- C-ABI mirror (same names)
def qr_birank_build(bits, n: int, device: int = 0, stream=None) -> Index:
    _need(bits, 8, (n + 63) // 64, "qr_birank_build bits")
    out = C.c_void_p()
    _check(lib().qr_birank_build(_ptr(bits), n, device, _stream(stream), C.byref(out)), "qr_birank_build")
    return Index(out.value)


def qr_build(text, n: int, layout: int, device: int = 0, stream=None) -> Index:
    sigma2 = layout in (QR_LAYOUT_BIRANK16, QR_LAYOUT_BIRANK64X2, QR_LAYOUT_BIRANK16X2, QR_LAYOUT_BIRANK32X2)
    _need(text, 8, (n + 63) // 64 if sigma2 else (n + 31) // 32, "qr_build text")
    out = C.c_void_p()
    _check(lib().qr_build(_ptr(text), n, layout, device, _stream(stream), C.byref(out)), "qr_build")
    return Index(out.value)


def qr_quadrank_build(text2b, n: int, device: int = 0, stream=None) -> Index:
    _need(text2b, 8, (n + 31) // 32, "qr_quadrank_build text2b")
    out = C.c_void_p()
    _check(lib().qr_quadrank_build(_ptr(text2b), n, device, _stream(stream), C.byref(out)), "qr_quadrank_build")
    return Index(out.value)


def qr_rank(h: Index, q, c, out, m: int | None = None, stream=None):
    m = (q.numel() if hasattr(q, "numel") else q.size) if m is None else m
    _need(q, 8, m, "qr_rank q")
    _need(out, 8, m, "qr_rank out")
    if c is not None:
        _need(c, 1, m, "qr_rank c")
    _check(lib().qr_rank(h.ptr, _ptr(q), _ptr(c), _ptr(out), m, _stream(stream)), "qr_rank")
    return out


def qr_rank_chain(h: Index, q, c, out, chain_len: int, m: int | None = None, stream=None):
    m = (q.numel() if hasattr(q, "numel") else q.size) if m is None else m
    _need(q, 8, m, "qr_rank_chain q")
    _need(out, 8, m, "qr_rank_chain out")
    if c is not None:
        _need(c, 1, m, "qr_rank_chain c")
    _check(lib().qr_rank_chain(h.ptr, _ptr(q), _ptr(c), _ptr(out), m, chain_len, _stream(stream)), "qr_rank_chain")
    return out


def qr_rank_all4(h: Index, q, out4, m: int | None = None, stream=None):
    m = (q.numel() if hasattr(q, "numel") else q.size) if m is None else m
    _need(q, 8, m, "qr_rank_all4 q")
    _need(out4, 8, 4 * m, "qr_rank_all4 out4")
    _check(lib().qr_rank_all4(h.ptr, _ptr(q), _ptr(out4), m, _stream(stream)), "qr_rank_all4")
    return out4


def qr_fm_build(text2b, n: int, sa=None, device: int = 0, stream=None, kmer_k: int | None = None,
                bwt_layout: int | None = None) -> Fm:
    """qr_fm_build (kmer_k None: the library's default width for n), qr_fm_build_ex (explicit width) or
    qr_fm_build_opts (explicit BWT rank layout, QR_LAYOUT_QUADRANK16 or QR_LAYOUT_QUADRANK16X2)."""
    _need(text2b, 8, (n + 31) // 32, "qr_fm_build text2b")
    _need(sa, 4, n + 1, "qr_fm_build sa")
    out = C.c_void_p()
    if bwt_layout is not None:
        k = kmer_k if kmer_k is not None else -1          # -1: the library's default width for n
        _check(lib().qr_fm_build_opts(_ptr(text2b), n, _ptr(sa), k, bwt_layout, device, _stream(stream), C.byref(out)),
               "qr_fm_build_opts")
        return Fm(out.value)
    if kmer_k is None:
        _check(lib().qr_fm_build(_ptr(text2b), n, _ptr(sa), device, _stream(stream), C.byref(out)), "qr_fm_build")
    else:
        _check(lib().qr_fm_build_ex(_ptr(text2b), n, _ptr(sa), kmer_k, device, _stream(stream), C.byref(out)),
               "qr_fm_build_ex")
    return Fm(out.value)


def qr_fm_build_u8(text, n: int, sa=None, device: int = 0, stream=None) -> Fm:
    """QuadFm index from one byte per symbol (0..3), packed on the GPU (SURVEY §8(b) input form)."""
    _need(text, 1, n, "qr_fm_build_u8 text")
    _need(sa, 4, n + 1, "qr_fm_build_u8 sa")
    out = C.c_void_p()
    _check(lib().qr_fm_build_u8(_ptr(text), n, _ptr(sa), device, _stream(stream), C.byref(out)), "qr_fm_build_u8")
    return Fm(out.value)


def _need_fm(where: str, patterns, lengths, fixed_len: int, m: int, *outs):
    for o in outs:
        _need(o, 4, m, f"{where} out")
    if lengths is not None:
        _need(lengths, 4, m, f"{where} lengths")
        _contig(patterns, f"{where} patterns")
    else:
        _need(patterns, 1, m * fixed_len, f"{where} patterns")


def qr_fm_count(fm: Fm, patterns, lengths, fixed_len: int, out, m: int, stream=None):
    _need_fm("qr_fm_count", patterns, lengths, fixed_len, m, out)
    _check(lib().qr_fm_count(fm.ptr, _ptr(patterns), _ptr(lengths), fixed_len, _ptr(out), m, _stream(stream)),
           "qr_fm_count")
    return out


def qr_fm_count_both(fm: Fm, patterns, lengths, fixed_len: int, out_fwd, out_rc, m: int, stream=None):
    _need_fm("qr_fm_count_both", patterns, lengths, fixed_len, m, out_fwd, out_rc)
    _check(lib().qr_fm_count_both(fm.ptr, _ptr(patterns), _ptr(lengths), fixed_len, _ptr(out_fwd), _ptr(out_rc), m,
                                  _stream(stream)), "qr_fm_count_both")
    return out_fwd, out_rc


def qr_fm_count_approx(fm: Fm, patterns, lengths, fixed_len: int, max_mismatches: int, out, m: int, stream=None):
    _need_fm("qr_fm_count_approx", patterns, lengths, fixed_len, m, out)
    _check(lib().qr_fm_count_approx(fm.ptr, _ptr(patterns), _ptr(lengths), fixed_len, max_mismatches, _ptr(out), m,
                                    _stream(stream)), "qr_fm_count_approx")
    return out


def qr_fm_count_approx_both(fm: Fm, patterns, lengths, fixed_len: int, max_mismatches: int, out_fwd, out_rc, m: int,
                            stream=None):
    _need_fm("qr_fm_count_approx_both", patterns, lengths, fixed_len, m, out_fwd, out_rc)
    _check(lib().qr_fm_count_approx_both(fm.ptr, _ptr(patterns), _ptr(lengths), fixed_len, max_mismatches,
                                         _ptr(out_fwd), _ptr(out_rc), m, _stream(stream)), "qr_fm_count_approx_both")
    return out_fwd, out_rc


def qr_fm_count_work(fm: Fm, patterns, lengths, fixed_len: int, out, m: int, work, stream=None):
    _need_fm("qr_fm_count_work", patterns, lengths, fixed_len, m, out)
    _need(work, 8, 2, "qr_fm_count_work work")
    _check(lib().qr_fm_count_work(fm.ptr, _ptr(patterns), _ptr(lengths), fixed_len, _ptr(out), m, _ptr(work),
                                  _stream(stream)), "qr_fm_count_work")
    return out


def qr_fm_count_work_ex(fm: Fm, patterns, lengths, fixed_len: int, max_mismatches: int, out, out_rc, m: int, work,
                        stream=None):
    """Work accounting of any count flavour (exact or <= 3 substitutions, one or both strands):
    work[0] += rank evaluations at interval ends + table lookups, work[1] += lines gathered."""
    if out_rc is None:
        _need_fm("qr_fm_count_work_ex", patterns, lengths, fixed_len, m, out)
    else:
        _need_fm("qr_fm_count_work_ex", patterns, lengths, fixed_len, m, out, out_rc)
    _need(work, 8, 2, "qr_fm_count_work_ex work")
    _check(lib().qr_fm_count_work_ex(fm.ptr, _ptr(patterns), _ptr(lengths), fixed_len, max_mismatches, _ptr(out),
                                     _ptr(out_rc), m, _ptr(work), _stream(stream)), "qr_fm_count_work_ex")
    return out


def qr_gather_ceiling(h: Index, q, out, mode: int = 0, m: int | None = None, stream=None):
    m = (q.numel() if hasattr(q, "numel") else q.size) if m is None else m
    _need(q, 8, m, "qr_gather_ceiling q")
    _need(out, 8, 4 * m if mode == 4 else m, "qr_gather_ceiling out")
    _check(lib().qr_gather_ceiling(h.ptr, _ptr(q), _ptr(out), m, mode, _stream(stream)), "qr_gather_ceiling")
    return out


def qr_export_layout(h: Index):
    import numpy as np

    lines = np.empty(h.line_bytes, dtype=np.uint8)
    sup = np.empty(h.super_bytes, dtype=np.uint8)
    _check(lib().qr_export_layout(h.ptr, _ptr(lines), _ptr(sup)), "qr_export_layout")
    return lines, sup.view(np.uint32)


def _byte_size(a) -> int:
    if a is None:
        return 0
    es, n = _nbytes_item(a)
    return es * n


def qr_import_layout(lines, sup, n: int, layout: int, device: int = 0, stream=None) -> Index:
    """lines / sup: contiguous torch tensors or numpy arrays (host or device) holding exactly the
    layout's bytes; their sizes are passed to the library, which rejects a mismatch."""
    _contig(lines, "qr_import_layout lines")
    if sup is not None and _byte_size(sup) == 0:
        sup = None
    _contig(sup, "qr_import_layout super")
    out = C.c_void_p()
    _check(lib().qr_import_layout(_ptr(lines), _byte_size(lines), _ptr(sup), _byte_size(sup), n, layout, device,
                                  _stream(stream), C.byref(out)), "qr_import_layout")
    return Index(out.value)


def save_index(h: Index, path: str):
    """Write a layout to a .npz file (header: n, layout; arrays: lines, super)."""
    import numpy as np

    lines, sup = qr_export_layout(h)
    np.savez(path, n=np.uint64(h.n), layout=np.int32(h.layout), lines=lines, super=sup)


def load_index(path: str, device: int = 0) -> Index:
    import numpy as np

    z = np.load(path)
    return qr_import_layout(np.ascontiguousarray(z["lines"]), np.ascontiguousarray(z["super"]), int(z["n"]),
                            int(z["layout"]), device)


def qr_fm_export_kmer(fm: Fm):
    import numpy as np

    ne = 1 << (2 * fm.kmer_k)
    t = np.empty(2 * ne, dtype=np.uint32)
    _check(lib().qr_fm_export_kmer(fm.ptr, _ptr(t)), "qr_fm_export_kmer")
    return t.reshape(ne, 2)


def qr_clone_to_device(h: Index, device: int, stream=None) -> Index:
    out = C.c_void_p()
    _check(lib().qr_clone_to_device(h.ptr, device, _stream(stream), C.byref(out)), "qr_clone_to_device")
    return Index(out.value)


def qr_fm_clone_to_device(fm: Fm, device: int, stream=None) -> Fm:
    out = C.c_void_p()
    _check(lib().qr_fm_clone_to_device(fm.ptr, device, _stream(stream), C.byref(out)), "qr_fm_clone_to_device")
    return Fm(out.value)


def qr_super_cache_bytes(h: "Index") -> int:
    """Shared-memory bytes per CTA of the superblock table the rank kernels use (0 = none)."""
    v = C.c_uint64(0)
    _check(lib().qr_super_cache_bytes(h.ptr, C.byref(v)), "qr_super_cache_bytes")
    return int(v.value)


def qr_super_cache_clusters(h: "Index") -> int:
    """2-CTA clusters the shared-memory rank kernels launch (0 = no table)."""
    v = C.c_int(0)
    _check(lib().qr_super_cache_clusters(h.ptr, C.byref(v)), "qr_super_cache_clusters")
    return int(v.value)


def qr_checksum(data, count: int, word_bytes: int, index0: int, acc, stream=None):
    """acc (1 u64 on the device) += sum_i mix(index0 + i, data[i]) mod 2^64: additive over shards."""
    _need(data, word_bytes, count, "qr_checksum data")
    _need(acc, 8, 1, "qr_checksum acc")
    _check(lib().qr_checksum(_ptr(data), count, word_bytes, index0, _ptr(acc), _stream(stream)), "qr_checksum")
    return acc


def qr_sync(stream=None):
    _check(lib().qr_sync(_stream(stream)), "qr_sync")


def qr_set_tuning(key: str, value: int):
    _check(lib().qr_set_tuning(key.encode(), int(value)), "qr_set_tuning")


def qr_version() -> str:
    return lib().qr_version().decode()


lib()  # fail loudly at import when the native library is missing
