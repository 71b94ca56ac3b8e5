"""Random-gather saturation: BiRank16 cluster rank kernel (configs[1]) and its load-only ceiling
(mode 3) vs the number of SMs used (2-CTA clusters, one CTA per SM).  A memory-side limit shows
as throughput that stops growing well before all 148 SMs are in use."""
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
M = 4 * 10**8
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n); del bits
q = torch.empty(M, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, M, q); out = torch.empty_like(q)
full = qr.qr_super_cache_clusters(h)
for ncl in (4, 8, 16, 24, 32, 40, 48, 56, 64, 74):
    if ncl > full: continue
    qr.qr_set_tuning("rank_smem_clusters", ncl)
    r = {"clusters": ncl, "sms": 2 * ncl}
    r["rank_gq_s"] = M / t(lambda: qr.qr_rank(h, q, None, out, M, st)) / 1e6
    r["ceil3_gq_s"] = M / t(lambda: qr.qr_gather_ceiling(h, q, out, 3, M, st)) / 1e6
    r["per_sm_mq_s"] = r["rank_gq_s"] * 1e3 / (2 * ncl)
    print(json.dumps(r), flush=True)
qr.qr_set_tuning("rank_smem_clusters", 0)
