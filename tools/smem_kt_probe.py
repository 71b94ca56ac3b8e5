"""Cluster rank kernels: (K, CTA threads) sweep on configs[1] (BiRank16) and configs[2] (QuadRank16
rank, rank_4), dynamic order; results compared with the global-memory kernels."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
KT = [(2, 1024), (3, 1024), (4, 1024), (4, 768), (6, 768), (8, 512)]
M = 10**9
def setkt(k, th):
    qr.qr_set_tuning("rank_smem_k", k); qr.qr_set_tuning("rank_smem_threads", th)
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n); del bits
q = torch.empty(M, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, M, q); out = torch.empty_like(q)
ref = torch.empty_like(q)
qr.qr_set_tuning("rank_smem", 0); qr.qr_rank(h, q, None, ref, M, st); qr.qr_set_tuning("rank_smem", 2)
for k, th in KT:
    setkt(k, th)
    r = {"kernel": "bi", "K": k, "threads": th, "gq_s": M / t(lambda: qr.qr_rank(h, q, None, out, M, st)) / 1e6}
    torch.cuda.synchronize(); r["equal"] = bool(torch.equal(out, ref)); print(json.dumps(r), flush=True)
del ref; h.free(); torch.cuda.empty_cache()
n = 1 << 32
text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, text)
h = qr.qr_quadrank_build(text, n); del text
c = torch.empty(M, dtype=torch.uint8, device=dev); gen.queries_dev(3, n, M, q, c)
ref = torch.empty_like(q)
qr.qr_set_tuning("rank_smem", 0); qr.qr_rank(h, q, c, ref, M, st); qr.qr_set_tuning("rank_smem", 2)
for k, th in KT:
    setkt(k, th)
    r = {"kernel": "qd_rank", "K": k, "threads": th, "gq_s": M / t(lambda: qr.qr_rank(h, q, c, out, M, st)) / 1e6}
    torch.cuda.synchronize(); r["equal"] = bool(torch.equal(out, ref)); print(json.dumps(r), flush=True)
del ref, out
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev); r4 = torch.empty_like(o4)
qr.qr_set_tuning("rank_smem", 0); qr.qr_rank_all4(h, q, r4, M, st); qr.qr_set_tuning("rank_smem", 2)
for k, th in KT:
    setkt(k, th)
    r = {"kernel": "qd_all4", "K": k, "threads": th, "gq_s": M / t(lambda: qr.qr_rank_all4(h, q, o4, M, st)) / 1e6}
    torch.cuda.synchronize(); r["equal"] = bool(torch.equal(o4, r4)); print(json.dumps(r), flush=True)
qr.qr_set_tuning("rank_smem_k", 0); qr.qr_set_tuning("rank_smem", 1)
