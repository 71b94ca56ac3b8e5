"""configs[0]-sized structures (2^20 bits; 2^19 DNA chars) at 10^6 queries: resident (lines in
every CTA's shared memory) vs lines from L2, rank / rank with c / QuadRank rank / rank_4."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=20):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for n in (1 << 20, 1 << 17, 1_400_000):
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(1, n, 0.5, bits)
    h = qr.qr_birank_build(bits, n)
    n4 = n // 2
    txt = torch.empty((n4 + 31) // 32 + 1, dtype=torch.uint64, device=dev); gen.dna_dev(3, n4, 0, txt)
    h4 = qr.qr_quadrank_build(txt, n4)
    for m in (10**6, 10**7):
        q = torch.empty(m, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, m, q)
        q4 = torch.empty(m, dtype=torch.uint64, device=dev); c4 = torch.empty(m, dtype=torch.uint8, device=dev)
        gen.queries_dev(3, n4, m, q4, c4)
        out = torch.empty_like(q); o4 = torch.empty((m, 4), dtype=torch.uint64, device=dev)
        for res in (1, 0):
            qr.qr_set_tuning("rank_resident", res)
            r = {"n": n, "m": m, "resident": res}
            r["bi_gq_s"] = m / t(lambda: qr.qr_rank(h, q, None, out, m, st)) / 1e6
            r["qd_gq_s"] = m / t(lambda: qr.qr_rank(h4, q4, c4, out, m, st)) / 1e6
            r["qd4_gq_s"] = m / t(lambda: qr.qr_rank_all4(h4, q4, o4, m, st)) / 1e6
            print(json.dumps(r), flush=True)
        qr.qr_set_tuning("rank_resident", 1)
