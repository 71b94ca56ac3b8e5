"""A/B of the cluster shared-memory superblock kernels (sbcache.cu) vs the global-memory lane-pair
kernels on configs[1] (BiRank16, n = 2^34, 10^9 q) and configs[2] (QuadRank16, n = 2^32, 10^9 (q,c)),
with the gather ceilings beside them; parity of the two paths on the full batch."""
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
h = qr.qr_birank_build(bits, n); del bits
print(json.dumps({"bi_cache_cta_bytes": qr.qr_super_cache_bytes(h)}), flush=True)
q = torch.empty(M, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, M, q); out = torch.empty_like(q)
out0 = torch.empty_like(q)
qr.qr_set_tuning("rank_smem", 0); qr.qr_rank(h, q, None, out0, M, st)
for k in ([4] if ONCE else [4, 2, 6, 8]):
    qr.qr_set_tuning("rank_smem_k", k)
    r = {"kernel": "bi", "K": k}
    for sm, dyn in ((0, 0), (2, 0), (2, 1)):
        qr.qr_set_tuning("rank_smem", sm); qr.qr_set_tuning("rank_dyn", dyn)
        r[f"rank_smem{sm}_dyn{dyn}"] = M / t(lambda: qr.qr_rank(h, q, None, out, M, st)) / 1e6
        torch.cuda.synchronize()
        r[f"equal_smem{sm}_dyn{dyn}"] = bool(torch.equal(out, out0))
    if not ONCE:
        for mode, dyn in ((0, 0), (2, 0), (3, 0), (3, 1)):
            qr.qr_set_tuning("rank_dyn", dyn)
            r[f"ceil{mode}_dyn{dyn}"] = M / t(lambda: qr.qr_gather_ceiling(h, q, out, mode, M, st)) / 1e6
    qr.qr_set_tuning("rank_dyn", 0)
    print(json.dumps(r), flush=True)
qr.qr_set_tuning("rank_smem_k", 4)
del q, out, out0; h.free(); torch.cuda.empty_cache()
n = 1 << 32
text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, text)
h = qr.qr_quadrank_build(text, n); del text
print(json.dumps({"qd_cache_cta_bytes": qr.qr_super_cache_bytes(h)}), flush=True)
q = torch.empty(M, dtype=torch.uint64, device=dev); c = torch.empty(M, dtype=torch.uint8, device=dev)
gen.queries_dev(3, n, M, q, c); out = torch.empty_like(q); out0 = torch.empty_like(q)
qr.qr_set_tuning("rank_smem", 0); qr.qr_rank(h, q, c, out0, M, st)
r = {"kernel": "qd"}
for sm, k in ((0, 4), (2, 2), (2, 4), (2, 6), (2, 8)):
    qr.qr_set_tuning("rank_smem", sm); qr.qr_set_tuning("rank_smem_k", k)
    r[f"rank_smem{sm}_k{k}"] = M / t(lambda: qr.qr_rank(h, q, c, out, M, st)) / 1e6
    torch.cuda.synchronize(); r[f"equal_smem{sm}_k{k}"] = bool(torch.equal(out, out0))
if not ONCE:
    r["ceil0"] = M / t(lambda: qr.qr_gather_ceiling(h, q, out, 0, M, st)) / 1e6
del out, out0
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev); o40 = torch.empty_like(o4)
qr.qr_set_tuning("rank_smem", 0); qr.qr_rank_all4(h, q, o40, M, st)
for sm, k in ((0, 4), (2, 2), (2, 4), (2, 6), (2, 8)):
    qr.qr_set_tuning("rank_smem", sm); qr.qr_set_tuning("rank_smem_k", k)
    r[f"all4_smem{sm}_k{k}"] = M / t(lambda: qr.qr_rank_all4(h, q, o4, M, st)) / 1e6
    torch.cuda.synchronize(); r[f"all4_equal_smem{sm}_k{k}"] = bool(torch.equal(o4, o40))
print(json.dumps(r), flush=True)
