"""n = 2^34 bits, 10^9 queries: the 2-CTA table kernel vs the large-n table forced at cluster size
4 / 8 / 16 (isolates the cluster-size cost from the size of the bit vector)."""
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
n, m = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 34), 10**9
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(1, n, 0.5, bits)
q = torch.empty(m, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, m, q)
out = torch.empty_like(q)
for cs in (0, 4, 8, 16):
    qr.qr_set_tuning("rank_big_pack", 1 if cs else 0)
    qr.qr_set_tuning("rank_big_cs", cs)
    h = qr.qr_birank_build(bits, n)
    qr.qr_set_tuning("rank_big_pack", 0); qr.qr_set_tuning("rank_big_cs", 0)
    ms = t(lambda: qr.qr_rank(h, q, None, out, m, st))
    print(json.dumps({"cs": cs, "ms": ms, "gq_s": m / ms / 1e6, "checksum": int(out[:1000000].sum())}), flush=True)
    del h
