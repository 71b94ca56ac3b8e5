"""One resident and one L2 launch of BiRank rank on 2^20 bits with 10^7 queries (ncu driver)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
n, m = 1 << 20, 10**7
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(1, n, 0.5, bits)
h = qr.qr_birank_build(bits, n)
q = torch.empty(m, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, m, q)
out = torch.empty_like(q)
for res in (1, 0):
    qr.qr_set_tuning("rank_resident", res)
    qr.qr_rank(h, q, None, out, m, st)
torch.cuda.synchronize()
print("ok")
