"""A/B of the lane-pair BiRank rank kernel vs its ceilings (with / without the superblock load)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
ONCE = len(sys.argv) > 1 and sys.argv[1] == "once"
def t(fn, reps=5):
    if ONCE:
        fn(); torch.cuda.synchronize(); return 1.0
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
n, M = 1 << 34, 10**9
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n); del bits
q = torch.empty(M, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, M, q); out = torch.empty_like(q)
for k, bps in ([(2, 64)] if ONCE else [(2, 64), (2, 32), (4, 64), (1, 64), (1, 128)]):
    qr.qr_set_tuning("rank_k", k); qr.qr_set_tuning("rank_blocks_per_sm", bps)
    r = {}
    for sl in (0, 1):
        qr.qr_set_tuning("rank_s_lane", sl)
        r[f"rank_s{sl}"] = M / t(lambda: qr.qr_rank(h, q, None, out, M, st)) / 1e6
    qr.qr_set_tuning("rank_s_lane", 0)
    for mode in (0, 2):
        r[f"ceil{mode}"] = M / t(lambda: qr.qr_gather_ceiling(h, q, out, mode, M, st)) / 1e6
    print(json.dumps(dict(K=k, bps=bps, **r)), flush=True)
