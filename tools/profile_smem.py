"""One launch each of the cluster shared-memory rank kernels (sbcache.cu) and of the global-memory
lane-pair kernels they replace, on configs[1] / configs[2] structures with 2*10^8 queries, for
ncu --set full captures.  Order: bi_rank2 (global), bi_rank2c (K=4, dyn), qd_rank2 (global),
qd_rank2c (K=2, dyn), qd_all4_2 (global), qd_all4_2c (K=2, dyn)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
M = 2 * 10**8
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev)
gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n)
del bits
q = torch.empty(M, dtype=torch.uint64, device=dev)
gen.queries_dev(2, n, M, q)
out = torch.empty_like(q)
qr.qr_set_tuning("rank_smem", 0)
qr.qr_rank(h, q, None, out, M, st)
qr.qr_set_tuning("rank_smem", 2)
qr.qr_set_tuning("rank_smem_k", 4)
qr.qr_rank(h, q, None, out, M, st)
torch.cuda.synchronize()
h.free()
n4 = 1 << 32
t = torch.empty((n4 + 31) // 32, dtype=torch.uint64, device=dev)
gen.dna_dev(3, n4, 0, t)
h = qr.qr_quadrank_build(t, n4)
del t
c = torch.empty(M, dtype=torch.uint8, device=dev)
gen.queries_dev(3, n4, M, q, c)
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev)
qr.qr_set_tuning("rank_smem_k", 2)
for sm in (0, 2):
    qr.qr_set_tuning("rank_smem", sm)
    qr.qr_rank(h, q, c, out, M, st)
for sm in (0, 2):
    qr.qr_set_tuning("rank_smem", sm)
    qr.qr_rank_all4(h, q, o4, M, st)
torch.cuda.synchronize()
print("ok")
