"""Near the 2-CTA table's capacity (parts 200-227 KB): BiRank16 at n = 1.23 x 2^34 bits and
QuadRank16 at n = 1.45 x 2^32 chars, 2-CTA table vs the CS-CTA table forced (rank_big_pack)."""
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
q = torch.empty(m, dtype=torch.uint64, device=dev); out = torch.empty_like(q)
c = torch.empty(m, dtype=torch.uint8, device=dev)
nb = int(1.23 * (1 << 34))
bits = torch.empty((nb + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(1, nb, 0.5, bits)
gen.queries_dev(2, nb, m, q)
for big in (0, 1):
    qr.qr_set_tuning("rank_big_pack", big)
    h = qr.qr_birank_build(bits, nb)
    qr.qr_set_tuning("rank_big_pack", 0)
    ms = t(lambda: qr.qr_rank(h, q, None, out, m, st))
    print(json.dumps({"sigma": 2, "n": nb, "big": big, "part_kb": qr.qr_super_cache_bytes(h) / 1024, "gq_s": m / ms / 1e6}), flush=True)
    del h
del bits; torch.cuda.empty_cache()
n4 = int(1.45 * (1 << 32))
txt = torch.empty((n4 + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n4, 0, txt)
gen.queries_dev(3, n4, m, q, c)
for big in (0, 1):
    qr.qr_set_tuning("rank_big_pack", big)
    h = qr.qr_quadrank_build(txt, n4)
    qr.qr_set_tuning("rank_big_pack", 0)
    ms = t(lambda: qr.qr_rank(h, q, c, out, m, st))
    print(json.dumps({"sigma": 4, "n": n4, "big": big, "part_kb": qr.qr_super_cache_bytes(h) / 1024, "gq_s": m / ms / 1e6}), flush=True)
    del h
