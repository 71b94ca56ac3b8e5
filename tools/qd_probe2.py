"""Per-launch times of the cluster rank kernels (diagnostic of launch-to-launch variance)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def each(fn, reps=12):
    fn(); torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(st)
    for i in range(reps):
        fn(); ev[i + 1].record(st)
    torch.cuda.synchronize()
    return [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(reps)]
n = 1 << 32
M = 10**9
text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n, 0, text)
h = qr.qr_quadrank_build(text, n); del text
print(json.dumps({"clusters": qr.qr_super_cache_clusters(h), "cta_bytes": qr.qr_super_cache_bytes(h)}), flush=True)
q = torch.empty(M, dtype=torch.uint64, device=dev); c = torch.empty(M, dtype=torch.uint8, device=dev)
gen.queries_dev(3, n, M, q, c); out = torch.empty_like(q)
for sm, k, dyn, ncl in ((0, 4, 1, 0), (2, 2, 1, 0), (2, 4, 1, 0), (2, 2, 1, 64), (2, 2, 1, 70), (2, 4, 1, 64), (2, 2, 0, 0)):
    qr.qr_set_tuning("rank_smem", sm); qr.qr_set_tuning("rank_smem_k", k); qr.qr_set_tuning("rank_dyn", dyn)
    qr.qr_set_tuning("rank_smem_clusters", ncl)
    print(json.dumps({"smem": sm, "k": k, "dyn": dyn, "clusters": ncl, "ms": each(lambda: qr.qr_rank(h, q, c, out, M, st))}), flush=True)
