"""Kernel-shape crossover vs structure size: one lane per query (global s), lane pairs (global s,
dynamic order), lane pairs with cluster shared-memory s; 2*10^8 uniform queries per point."""
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
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev)
SH = [("lane", 1, 0, 0), ("lane_table", 1, 0, 1), ("pair", 0, 1, 1), ("cluster", 2, 1, 1), ("auto", 1, 2, 1)]
def run(h, cc, r):
    for name, smem, pair, lt in SH:
        qr.qr_set_tuning("rank_smem", smem); qr.qr_set_tuning("rank_pair", pair); qr.qr_set_tuning("rank_lane_table", lt)
        r[name] = round(M / t(lambda: qr.qr_rank(h, q, cc, out, M, st)) / 1e6, 2)
        if cc is not None:
            r[name + "_all4"] = round(M / t(lambda: qr.qr_rank_all4(h, q, o4, M, st)) / 1e6, 2)
for lg in (24, 26, 28, 29, 30, 31, 32, 34):
    n = 1 << lg
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(7, n, 0.5, bits)
    h = qr.qr_birank_build(bits, n); del bits
    gen.queries_dev(8, n, M, q)
    r = {"sigma": 2, "log2_n": lg, "line_mb": round(h.line_bytes / 2**20, 1)}
    run(h, None, r)
    print(json.dumps(r), flush=True)
    h.free(); torch.cuda.empty_cache()
for lg in (24, 26, 27, 28, 29, 30, 32):
    n = 1 << lg
    text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(9, n, 0, text)
    h = qr.qr_quadrank_build(text, n); del text
    gen.queries_dev(10, n, M, q, c)
    r = {"sigma": 4, "log2_n": lg, "line_mb": round(h.line_bytes / 2**20, 1)}
    run(h, c, r)
    print(json.dumps(r), flush=True)
    h.free(); torch.cuda.empty_cache()
qr.qr_set_tuning("rank_smem", 1); qr.qr_set_tuning("rank_pair", 2); qr.qr_set_tuning("rank_lane_table", 1)
