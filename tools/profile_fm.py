"""One launch each of the QuadFm count kernel on configs[3] and configs[4] at the library defaults
(persistent warp-chunk order, default k-mer width), for ncu --set full captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
for n, kind, m, L, seed in ((1 << 26, 0, 10**7, 32, 4), (1 << 30, 1, 10**8, 100, 5)):
    t = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
    gen.dna_dev(seed, n, kind, t)
    fm = qr.qr_fm_build(t, n)
    pats = torch.empty(m * L, dtype=torch.uint8, device=dev)
    gen.patterns_dev(seed, kind, m, L, t, n, pats)
    o = torch.empty(m, dtype=torch.int32, device=dev)
    qr.qr_fm_count(fm, pats, None, L, o, m, st)
    torch.cuda.synchronize()
    fm.free()
    del t, pats, o
    torch.cuda.empty_cache()
print("ok")
