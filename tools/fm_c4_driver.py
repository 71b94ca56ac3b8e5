"""configs[3] QuadFm count, one launch per (BWT layout, fm_step flavour) after one warm-up call —
the command the ncu captures of the count and seed kernels run (FM_STEPS='16:2,16:3,x2:0,x2:3';
an item may add the k-mer width and the packed-seed knob: '16:3:11:0')."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
n, m, L = 1 << 26, 10**7, 32
t = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
gen.dna_dev(4, n, 0, t)
pats = torch.empty(m * L, dtype=torch.uint8, device=dev)
gen.patterns_dev(4, 0, m, L, t, n, pats)
o = torch.empty(m, dtype=torch.int32, device=dev)
plan = os.environ.get("FM_STEPS", "16:2,16:3,x2:0,x2:3").split(",")
fms = {}
for item in plan:
    f = item.split(":")
    lay, step = f[0], int(f[1])
    kk = int(f[2]) if len(f) > 2 else None
    packed = int(f[3]) if len(f) > 3 else 1
    key = (lay, kk)
    if key not in fms:
        fms[key] = qr.qr_fm_build(t, n, bwt_layout=qr.QR_LAYOUT_QUADRANK16 if lay == "16" else qr.QR_LAYOUT_QUADRANK16X2,
                                  kmer_k=kk)
    qr.qr_set_tuning("fm_step", step)
    qr.qr_set_tuning("fm_packed", packed)
    qr.qr_fm_count(fms[key], pats, None, L, o, m, st)
    torch.cuda.synchronize()
print("ok")
