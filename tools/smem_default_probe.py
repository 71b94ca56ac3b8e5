"""Cluster rank kernels at the library defaults (BiRank rank, QuadRank rank, rank_4), one line each."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
tag = sys.argv[1] if len(sys.argv) > 1 else ""
def t(fn, reps=5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
M = 10**9
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n); del bits
q = torch.empty(M, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, M, q); out = torch.empty_like(q)
r = {"tag": tag, "bi_rank": M / t(lambda: qr.qr_rank(h, q, None, out, M, st)) / 1e6,
     "bi_sum": int(out[:1000000].sum())}
h.free(); torch.cuda.empty_cache()
n = 1 << 32
text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, text)
h = qr.qr_quadrank_build(text, n); del text
c = torch.empty(M, dtype=torch.uint8, device=dev); gen.queries_dev(3, n, M, q, c)
r["qd_rank"] = M / t(lambda: qr.qr_rank(h, q, c, out, M, st)) / 1e6
del out
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev)
r["qd_all4"] = M / t(lambda: qr.qr_rank_all4(h, q, o4, M, st)) / 1e6
r["all4_sum"] = int(o4[:1000000].sum())
print(json.dumps(r), flush=True)
