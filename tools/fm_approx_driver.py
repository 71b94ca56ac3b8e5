"""configs[3] approximate counting (<= KMAX substitutions, 10^5 x 32) once per BWT layout — the
command the ncu captures of k_fm_approxk / k_fm_approx1 run (FM_KMAX=2, FM_M=100000).
FM_READS=1: the bench's 150-bp reads instead (configs[4] text, 2^30 symbols, both strands in one
launch, QuadRank16 BWT only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402

dev = torch.device("cuda:0")
reads = os.environ.get("FM_READS", "0") == "1"
n, L = (1 << 30, 150) if reads else (1 << 26, 32)
m = int(os.environ.get("FM_M", "100000"))
kmax = int(os.environ.get("FM_KMAX", "2"))
t = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
gen.dna_dev(5 if reads else 4, n, 1 if reads else 0, t)
pats = torch.empty(m * L, dtype=torch.uint8, device=dev)
gen.patterns_dev(55 if reads else 4, 2 if reads else 0, m, L, t, n, pats)
o = torch.empty(m, dtype=torch.int32, device=dev)
orc = torch.empty(m, dtype=torch.int32, device=dev)
for lay in ((qr.QR_LAYOUT_QUADRANK16,) if reads else (qr.QR_LAYOUT_QUADRANK16, qr.QR_LAYOUT_QUADRANK16X2)):
    fm = qr.qr_fm_build(t, n, bwt_layout=lay)
    if reads:
        qr.qr_fm_count_approx_both(fm, pats, None, L, kmax, o, orc, m)
    else:
        qr.qr_fm_count_approx(fm, pats, None, L, kmax, o, m)
    torch.cuda.synchronize()
    fm.free()
print("ok")
