"""Rank throughput vs structure size (the paper's throughput-vs-n view) for the
final default kernels: BiRank16 and BiRank64x2 over n = 2^20 .. 2^36 bits, QuadRank16 rank /
rank_4 and QuadRank64 rank over n = 2^20 .. 2^34 chars; 2*10^8 uniform queries per point."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=3):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
M = 2 * 10**8
q = torch.empty(M, dtype=torch.uint64, device=dev); out = torch.empty_like(q)
c = torch.empty(M, dtype=torch.uint8, device=dev)
for lg in ((20, 24, 26, 28, 30, 32, 34, 35, 36) if "dna_only" not in sys.argv else ()):
    n = 1 << lg
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(7, n, 0.5, bits)
    gen.queries_dev(8, n, M, q)
    r = {"sigma": 2, "log2_n": lg}
    for name, layout in (("birank16", qr.QR_LAYOUT_BIRANK16), ("birank16x2", qr.QR_LAYOUT_BIRANK16X2),
                         ("birank32x2", qr.QR_LAYOUT_BIRANK32X2), ("birank64x2", qr.QR_LAYOUT_BIRANK64X2)):
        h = qr.qr_build(bits, n, layout)
        r[name + "_gq_s"] = M / t(lambda: qr.qr_rank(h, q, None, out, M, st)) / 1e6
        r[name + "_bytes"] = h.line_bytes + h.super_bytes
        if layout == qr.QR_LAYOUT_BIRANK16:
            r["smem_cache"] = qr.qr_super_cache_bytes(h) > 0
        if layout == qr.QR_LAYOUT_BIRANK16X2:
            r["birank16x2_ceiling_gq_s"] = M / t(lambda: qr.qr_gather_ceiling(h, q, out, 0, M, st)) / 1e6
        h.free()
    del bits; torch.cuda.empty_cache()
    print(json.dumps(r), flush=True)
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev)
for lg in ((20, 24, 26, 28, 30, 32, 33, 34) if "bits_only" not in sys.argv else ()):
    n = 1 << lg
    text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(9, n, 0, text)
    gen.queries_dev(10, n, M, q, c)
    r = {"sigma": 4, "log2_n": lg}
    for name, layout in (("quadrank16", qr.QR_LAYOUT_QUADRANK16), ("quadrank16x2", qr.QR_LAYOUT_QUADRANK16X2),
                         ("quadrank64", qr.QR_LAYOUT_QUADRANK64)):
        h = qr.qr_build(text, n, layout)
        r[name + "_gq_s"] = M / t(lambda: qr.qr_rank(h, q, c, out, M, st)) / 1e6
        r[name + "_all4_gq_s"] = M / t(lambda: qr.qr_rank_all4(h, q, o4, M, st)) / 1e6
        r[name + "_bytes"] = h.line_bytes + h.super_bytes
        if layout == qr.QR_LAYOUT_QUADRANK16:
            r["smem_cache"] = qr.qr_super_cache_bytes(h) > 0
        h.free()
    del text; torch.cuda.empty_cache()
    print(json.dumps(r), flush=True)
