"""Approximate counting vs the k-mer table width (12 / 13 / 14) on configs[3] (10^6 x 32) and the
150-bp reads on the configs[4] text (both strands): patterns/s for k = 1, 2 (3 on configs[3], its first
2*10^5 patterns; APPROX_KMAX=1,2,3 picks) and the build time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
KMAXES = [int(x) for x in os.environ.get("APPROX_KMAX", "1,2").split(",")]


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name, n, kind, tseed, m, L, pk, pseed, both in (("c4", 1 << 26, 0, 4, 10**6, 32, 0, 4, False),
                                                    ("reads", 1 << 30, 1, 5, 3 * 10**5, 150, 2, 55, True)):
    txt = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
    gen.dna_dev(tseed, n, kind, txt)
    pats = torch.empty(m * L, dtype=torch.uint8, device=dev)
    gen.patterns_dev(pseed, pk, m, L, txt, n, pats)
    o = torch.empty(m, dtype=torch.int32, device=dev)
    orc = torch.empty(m, dtype=torch.int32, device=dev)
    for K in (12, 13, 14):
        t0 = time.perf_counter()
        fm = qr.qr_fm_build(txt, n, kmer_k=K)
        bs = time.perf_counter() - t0
        for kmax in KMAXES:
            mm = m if kmax < 3 else min(m, 2 * 10**5)
            if both and kmax == 3:
                continue
            if both:
                ms = t(lambda: qr.qr_fm_count_approx_both(fm, pats, None, L, kmax, o, orc, mm, st))
            else:
                ms = t(lambda: qr.qr_fm_count_approx(fm, pats, None, L, kmax, o, mm, st))
            print(json.dumps(dict(cfg=name, K=K, kmax=kmax, ms=round(ms, 3), per_s=mm / ms * 1e3, build_s=round(bs, 3),
                                  checksum=int(o[:mm].to(torch.int64).sum()))), flush=True)
        fm.free()
        torch.cuda.empty_cache()
