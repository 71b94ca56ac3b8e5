"""One launch each of the large-n cluster-table kernels (BiRank16 2^35 bits, QuadRank16 2^33
chars; 10^9 queries) for ncu captures."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
m = 10**9
n = 1 << 35
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(1, n, 0.5, bits)
h = qr.qr_birank_build(bits, n); del bits
q = torch.empty(m, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, m, q)
out = torch.empty_like(q)
qr.qr_rank(h, q, None, out, m, st); torch.cuda.synchronize()
del h
n4 = 1 << 33
txt = torch.empty((n4 + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(3, n4, 0, txt)
h4 = qr.qr_quadrank_build(txt, n4); del txt
c = torch.empty(m, dtype=torch.uint8, device=dev); gen.queries_dev(3, n4, m, q, c)
qr.qr_rank(h4, q, c, out, m, st); torch.cuda.synchronize()
print("ok")
