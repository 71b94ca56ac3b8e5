"""QuadRank16 rank / rank_4 at n = 2^32 chars (configs[2]), 10^9 queries: the 2-CTA table
(150 KB per CTA) vs the CS-CTA table forced at 4 / 8 CTAs (75 / 38 KB per CTA)."""
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
q = torch.empty(m, dtype=torch.uint64, device=dev); c = torch.empty(m, dtype=torch.uint8, device=dev)
gen.queries_dev(3, n, m, q, c)
out = torch.empty_like(q)
o4 = torch.empty((m // 4, 4), dtype=torch.uint64, device=dev)
for cs in (0, 4, 8):
    qr.qr_set_tuning("rank_big_pack", 1 if cs else 0); qr.qr_set_tuning("rank_big_cs", cs)
    h = qr.qr_quadrank_build(txt, n)
    qr.qr_set_tuning("rank_big_pack", 0); qr.qr_set_tuning("rank_big_cs", 0)
    ms = t(lambda: qr.qr_rank(h, q, c, out, m, st))
    ms4 = t(lambda: qr.qr_rank_all4(h, q[: m // 4], o4, m // 4, st))
    print(json.dumps({"cs": cs, "rank_gq_s": m / ms / 1e6, "all4_gq_s": m / 4 / ms4 / 1e6,
                      "checksum": int(out[:1000000].sum())}), flush=True)
    del h
