"""QuadRank cluster kernels: timing vs batch size and repetition (diagnostic)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=5, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
n = 1 << 32
MM = 10**9
text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, text)
h = qr.qr_quadrank_build(text, n); del text
q = torch.empty(MM, dtype=torch.uint64, device=dev); c = torch.empty(MM, dtype=torch.uint8, device=dev)
gen.queries_dev(3, n, MM, q, c); out = torch.empty_like(q)
for M in (2 * 10**8, 10**9):
    for sm, k, dyn in ((0, 4, 1), (2, 2, 1), (2, 2, 0), (2, 4, 1), (2, 1, 1)):
        qr.qr_set_tuning("rank_smem", sm); qr.qr_set_tuning("rank_smem_k", k); qr.qr_set_tuning("rank_dyn", dyn)
        r = {"M": M, "smem": sm, "k": k, "dyn": dyn}
        r["gq_s_loop"] = M / t(lambda: qr.qr_rank(h, q, c, out, M, st)) / 1e6
        r["gq_s_single"] = M / t(lambda: qr.qr_rank(h, q, c, out, M, st), reps=1, warm=1) / 1e6
        print(json.dumps(r), flush=True)
