"""One k_fm_count launch on configs[3] per BWT layout (QuadRank16, QuadRank16x2) for ncu metric
captures of the L1 / shared-memory wavefronts per backward step."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
n, m, L = 1 << 26, 10**7, 32
t = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
gen.dna_dev(4, n, 0, t)
pats = torch.empty(m * L, dtype=torch.uint8, device=dev)
gen.patterns_dev(4, 0, m, L, t, n, pats)
o = torch.empty(m, dtype=torch.int32, device=dev)
for lay in (qr.QR_LAYOUT_QUADRANK16, qr.QR_LAYOUT_QUADRANK16X2):
    fm = qr.qr_fm_build(t, n, bwt_layout=lay)
    qr.qr_fm_count(fm, pats, None, L, o, m, st)
    torch.cuda.synchronize()
    fm.free()
print("ok")
