"""Launch-grid sweep (K queries per thread x CTAs per SM) of the rank kernels on configs 2/3."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
M = 10**9
KS = [int(x) for x in os.environ.get("SWEEP_K", "2,4,8").split(",")]
BPS = [int(x) for x in os.environ.get("SWEEP_BPS", "4,8,16,32,64").split(",")]
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n); del bits
q = torch.empty(M, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, M, q); out = torch.empty_like(q)
PAIRS = [int(x) for x in os.environ.get("SWEEP_PAIR", "0,1").split(",")]
for pair in PAIRS:
  qr.qr_set_tuning("rank_pair", pair)
  for k in KS:
    for bps in BPS:
        qr.qr_set_tuning("rank_k", k); qr.qr_set_tuning("rank_blocks_per_sm", bps)
        ms = t(lambda: qr.qr_rank(h, q, None, out, M, st))
        g0 = t(lambda: qr.qr_gather_ceiling(h, q, out, 0, M, st))
        g1 = t(lambda: qr.qr_gather_ceiling(h, q, out, 1, M, st))
        print(json.dumps(dict(kernel="bi", pair=pair, K=k, bps=bps, gq_s=M / ms / 1e6, ceil0=M / g0 / 1e6, ceil1=M / g1 / 1e6)), flush=True)
h.free(); torch.cuda.empty_cache()
n = 1 << 32
txt = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, txt)
h = qr.qr_quadrank_build(txt, n); del txt
c = torch.empty(M, dtype=torch.uint8, device=dev); gen.queries_dev(3, n, M, q, c)
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev)
for pair in PAIRS:
  qr.qr_set_tuning("rank_pair", pair)
  for k in KS:
    for bps in BPS:
        qr.qr_set_tuning("rank_k", k); qr.qr_set_tuning("rank_blocks_per_sm", bps)
        ms = t(lambda: qr.qr_rank(h, q, c, out, M, st))
        m4 = t(lambda: qr.qr_rank_all4(h, q, o4, M, st))
        g0 = t(lambda: qr.qr_gather_ceiling(h, q, out, 0, M, st))
        print(json.dumps(dict(kernel="qd", pair=pair, K=k, bps=bps, gq_s=M / ms / 1e6, all4_gq_s=M / m4 / 1e6, ceil0=M / g0 / 1e6)), flush=True)
