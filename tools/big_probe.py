"""BiRank16 rank at 2^34 / 2^35 / 2^36 bits (10^9 uniform queries): default path (2-CTA table at
2^34, the 4/8-CTA cluster table beyond) vs rank_smem 0 (global lane-pair kernels)."""
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
for lg in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["34", "35", "36"])]:
    n = 1 << lg
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(1, n, 0.5, bits)
    h = qr.qr_birank_build(bits, n)
    del bits
    torch.cuda.empty_cache()
    q = torch.empty(m, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, m, q)
    out = torch.empty_like(q)
    for mode in (1, 0):
        qr.qr_set_tuning("rank_smem", mode)
        ms = t(lambda: qr.qr_rank(h, q, None, out, m, st))
        print(json.dumps({"n_log2": lg, "rank_smem": mode, "ms": ms, "gq_s": m / ms / 1e6,
                          "checksum": int(out[:1000000].sum())}), flush=True)
    qr.qr_set_tuning("rank_smem", 1)
    del h, q, out
    torch.cuda.empty_cache()
