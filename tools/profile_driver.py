"""One launch of each hot kernel at the bench's configs and default launch configuration, for
ncu --set full captures (kernel order: bi_rank2c (BiRank16 rank, cluster shared-memory superblocks),
BiRank16x2 / QuadRank16x2 rank (cluster kernels) after the QuadRank64 rank,
bi_gather2 x3 (ceiling modes 0-2), bi_rank2c<VAR=3> (ceiling mode 3), qd_rank2c, qd_all4_2c, b64_rank,
q64_rank, fm_count (c4, lean), fm_count (c5, de-duplicating), fm_count both strands, the breadth-first
<= 1 substitution on both strands of 10^6 reads, configs[3] <= 1 and <= 2 substitutions (breadth first)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
M = 10**9
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev)
gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n)
q = torch.empty(M, dtype=torch.uint64, device=dev)
gen.queries_dev(2, n, M, q)
out = torch.empty_like(q)
qr.qr_rank(h, q, None, out, M, st)
for mode in (0, 1, 2, 3):
    qr.qr_gather_ceiling(h, q, out, mode, M, st)
torch.cuda.synchronize()
h.free()
hb = qr.qr_build(bits, n, qr.QR_LAYOUT_BIRANK64X2)
hb16 = qr.qr_build(bits, n, qr.QR_LAYOUT_BIRANK16X2)
del bits
n4 = 1 << 32
t = torch.empty((n4 + 31) // 32, dtype=torch.uint64, device=dev)
gen.dna_dev(3, n4, 0, t)
h = qr.qr_quadrank_build(t, n4)
c = torch.empty(M, dtype=torch.uint8, device=dev)
gen.queries_dev(3, n4, M, q, c)
qr.qr_rank(h, q, c, out, M, st)
o4 = torch.empty((M, 4), dtype=torch.uint64, device=dev)
qr.qr_rank_all4(h, q, o4, M, st)
torch.cuda.synchronize()
h.free()
del o4
hq = qr.qr_build(t, n4, qr.QR_LAYOUT_QUADRANK64)
hq16 = qr.qr_build(t, n4, qr.QR_LAYOUT_QUADRANK16X2)
del t
qb = torch.empty(M, dtype=torch.uint64, device=dev)
gen.queries_dev(2, n, M, qb)
qr.qr_rank(hb, qb, None, out, M, st)
qr.qr_rank(hq, q, c, out, M, st)
qr.qr_rank(hb16, qb, None, out, M, st)
qr.qr_rank(hq16, q, c, out, M, st)
torch.cuda.synchronize()
hb.free(); hq.free(); hb16.free(); hq16.free()
del q, c, qb, out
n = 1 << 26
t = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
gen.dna_dev(4, n, 0, t)
fm = qr.qr_fm_build(t, n)
m = 10**7
pats = torch.empty(m * 32, dtype=torch.uint8, device=dev)
gen.patterns_dev(4, 0, m, 32, t, n, pats)
o = torch.empty(m, dtype=torch.int32, device=dev)
qr.qr_fm_count(fm, pats, None, 32, o, m, st)
torch.cuda.synchronize()
fm.free()
n = 1 << 30
t = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
gen.dna_dev(5, n, 1, t)
fm = qr.qr_fm_build(t, n)
m = 10**8
pats = torch.empty(m * 100, dtype=torch.uint8, device=dev)
gen.patterns_dev(5, 1, m, 100, t, n, pats)
o = torch.empty(m, dtype=torch.int32, device=dev)
qr.qr_fm_count(fm, pats, None, 100, o, m, st)
mr = 10**7
reads = torch.empty(mr * 150, dtype=torch.uint8, device=dev)
gen.patterns_dev(55, 2, mr, 150, t, n, reads)
of = torch.empty(mr, dtype=torch.int32, device=dev)
orc = torch.empty(mr, dtype=torch.int32, device=dev)
qr.qr_fm_count_both(fm, reads, None, 150, of, orc, mr, st)
torch.cuda.synchronize()
ma = 10**6                                   # <= 1 substitution on both strands (breadth first)
qr.qr_fm_count_approx_both(fm, reads[: ma * 150], None, 150, 1, of[:ma], orc[:ma], ma, st)
torch.cuda.synchronize()
fm.free()
n = 1 << 26
t = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
gen.dna_dev(4, n, 0, t)
fm = qr.qr_fm_build(t, n)
m = 10**6
pats = torch.empty(m * 32, dtype=torch.uint8, device=dev)
gen.patterns_dev(4, 0, m, 32, t, n, pats)
o = torch.empty(m, dtype=torch.int32, device=dev)
qr.qr_fm_count_approx(fm, pats, None, 32, 1, o, m, st)
qr.qr_fm_count_approx(fm, pats, None, 32, 2, o, m, st)
torch.cuda.synchronize()
print("profile driver done")
