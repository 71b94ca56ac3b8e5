"""QuadRank16 rank / rank_4 on configs[2] (2^32 chars, 10^9 queries): the 2-CTA cluster kernel's
(K, CTA threads) pairs."""
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
n, m = 1 << 32, 10**9
txt = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, txt)
h = qr.qr_quadrank_build(txt, n); del txt
q = torch.empty(m, dtype=torch.uint64, device=dev); c = torch.empty(m, dtype=torch.uint8, device=dev)
gen.queries_dev(3, n, m, q, c)
out = torch.empty_like(q)
o4 = torch.empty((m // 4, 4), dtype=torch.uint64, device=dev)
for k, th in ((2, 1024), (1, 1024), (3, 1024), (4, 1024), (4, 768), (6, 768), (8, 512)):
    qr.qr_set_tuning("rank_smem_k", k); qr.qr_set_tuning("rank_smem_threads", th)
    ms = t(lambda: qr.qr_rank(h, q, c, out, m, st))
    ms4 = t(lambda: qr.qr_rank_all4(h, q[: m // 4], o4, m // 4, st))
    print(json.dumps({"K": k, "threads": th, "rank_gq_s": m / ms / 1e6, "all4_gq_s": m / 4 / ms4 / 1e6}), flush=True)
qr.qr_set_tuning("rank_smem_k", 0)
