"""QuadRank16 rank / rank_4 at 2^32 / 2^33 / 2^34 chars (10^9 queries): default path (2-CTA table,
then the CS-CTA table) vs rank_smem 0 (global lane-pair kernels)."""
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
m = 10**9
for lg in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["32", "33", "34"])]:
    n = 1 << lg
    txt = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, txt)
    h = qr.qr_quadrank_build(txt, n)
    del txt
    torch.cuda.empty_cache()
    q = torch.empty(m, dtype=torch.uint64, device=dev); c = torch.empty(m, dtype=torch.uint8, device=dev)
    gen.queries_dev(3, n, m, q, c)
    out = torch.empty_like(q)
    for mode in (1, 0):
        qr.qr_set_tuning("rank_smem", mode)
        ms = t(lambda: qr.qr_rank(h, q, c, out, m, st))
        print(json.dumps({"n_log2": lg, "rank_smem": mode, "ms": ms, "gq_s": m / ms / 1e6,
                          "checksum": int(out[:1000000].sum())}), flush=True)
    qr.qr_set_tuning("rank_smem", 1)
    del h, q, c, out
    torch.cuda.empty_cache()
