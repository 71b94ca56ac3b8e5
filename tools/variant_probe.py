"""Layout variants (BiRank64x2, QuadRank64): static multi-wave vs persistent dynamic work order."""
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
M = 10**9
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_build(bits, n, qr.QR_LAYOUT_BIRANK64X2); del bits
q = torch.empty(M, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, M, q); out = torch.empty_like(q)
ref = torch.empty_like(q)
qr.qr_set_tuning("rank_dyn", 0); qr.qr_rank(h, q, None, ref, M, st)
for dyn in (0, 1):
    for k in (2, 4):
        qr.qr_set_tuning("rank_dyn", dyn); qr.qr_set_tuning("rank_k", k)
        r = {"layout": "birank64x2", "dyn": dyn, "K": k}
        r["rank_gq_s"] = M / t(lambda: qr.qr_rank(h, q, None, out, M, st)) / 1e6
        torch.cuda.synchronize(); r["equal"] = bool(torch.equal(out, ref))
        r["ceil_gq_s"] = M / t(lambda: qr.qr_gather_ceiling(h, q, out, 0, M, st)) / 1e6
        print(json.dumps(r), flush=True)
del ref; h.free(); torch.cuda.empty_cache()
n = 1 << 32
text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, text)
h = qr.qr_build(text, n, qr.QR_LAYOUT_QUADRANK64); del text
c = torch.empty(M, dtype=torch.uint8, device=dev); gen.queries_dev(3, n, M, q, c)
ref = torch.empty_like(q)
qr.qr_set_tuning("rank_dyn", 0); qr.qr_set_tuning("rank_k", 2); qr.qr_rank(h, q, c, ref, M, st)
for dyn in (0, 1):
    for k in (2, 4):
        qr.qr_set_tuning("rank_dyn", dyn); qr.qr_set_tuning("rank_k", k)
        r = {"layout": "quadrank64", "dyn": dyn, "K": k}
        r["rank_gq_s"] = M / t(lambda: qr.qr_rank(h, q, c, out, M, st)) / 1e6
        torch.cuda.synchronize(); r["equal"] = bool(torch.equal(out, ref))
        print(json.dumps(r), flush=True)
del out, ref
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev)
for dyn in (0, 1):
    qr.qr_set_tuning("rank_dyn", dyn); qr.qr_set_tuning("rank_k", 2)
    print(json.dumps({"layout": "quadrank64", "dyn": dyn, "K": 2,
                      "all4_gq_s": M / t(lambda: qr.qr_rank_all4(h, q, o4, M, st)) / 1e6}), flush=True)
qr.qr_set_tuning("rank_dyn", 1); qr.qr_set_tuning("rank_k", 2)
