"""One launch each of the newer kernels for ncu captures: resident small-structure rank (2^20 bits,
10^7 q), approximate search on both strands of 150-bp reads (k = 1, configs[4] text)."""
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
qr.qr_rank(h, q, None, out, m, st)
torch.cuda.synchronize()
del h, bits, q, out
n5, L, mr = 1 << 30, 150, 10**6
text = torch.empty((n5 + 31) // 32 + 1, dtype=torch.uint64, device=dev); gen.dna_dev(5, n5, 1, text)
fm = qr.qr_fm_build(text, n5)
pats = torch.empty(mr * L, dtype=torch.uint8, device=dev); gen.patterns_dev(55, 2, mr, L, text, n5, pats)
of = torch.empty(mr, dtype=torch.int32, device=dev); orc = torch.empty_like(of)
qr.qr_fm_count_approx_both(fm, pats, None, L, 1, of, orc, mr, st)
torch.cuda.synchronize()
print("ok")
