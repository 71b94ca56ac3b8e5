"""QuadFm count: step flavours (fm_step 1 de-dup, 2 lean, 3 one line per iteration) on configs[3]
and configs[4], both BWT layouts, next to the random-gather ceiling of the same BWT handle
(qr_gather_ceiling modes 0/1 on q uniform in [0, N]) — lines/s of the search vs lines/s the
memory system serves for that structure.  One JSON line per measurement."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream()


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


cfgs = [("c4", 1 << 26, 0, 10**7, 32, 4), ("c5", 1 << 30, 1, 10**8, 100, 5)]
if len(sys.argv) > 1:
    cfgs = [c for c in cfgs if c[0] in sys.argv[1].split(",")]
for name, n, kind, m, L, seed in cfgs:
    txt = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
    gen.dna_dev(seed, n, kind, txt)
    pats = torch.empty(m * L, dtype=torch.uint8, device=dev)
    gen.patterns_dev(seed, 0 if kind == 0 else 1, m, L, txt, n, pats)
    out = torch.empty(m, dtype=torch.int32, device=dev)
    ref = None
    for lay, lname in ((None, "qr16"), (qr.QR_LAYOUT_QUADRANK16X2, "qr16x2")):
        fm = qr.qr_fm_build(txt, n, bwt_layout=lay, kmer_k=int(os.environ["FM_K"]) if "FM_K" in os.environ else None)
        N = n + 1
        mq = 1 << 26
        q = torch.empty(mq, dtype=torch.uint64, device=dev)
        gen.queries_dev(seed + 100, N, mq, q)
        o = torch.empty(mq, dtype=torch.uint64, device=dev)
        ceil = {}
        for mode in (0, 1):
            ms = t(lambda: qr.qr_gather_ceiling(fm.bwt, q, o, mode, mq, st))
            ceil[mode] = mq / ms / 1e6
        c4 = torch.empty(mq, dtype=torch.uint8, device=dev)
        gen.queries_dev(seed + 101, N, mq, q, c4)
        ms = t(lambda: qr.qr_rank(fm.bwt, q, c4, o, mq, st))
        rank_gq = mq / ms / 1e6
        print(json.dumps(dict(cfg=name, layout=lname, kmer_k=fm.kmer_k, bwt_bytes=fm.bwt.line_bytes, ceiling_gq_s=ceil,
                              rank_gq_s=rank_gq)), flush=True)
        del q, o, c4
        steps = (1, 2, 3) if lay is None else (0, 3)
        refills = [int(x) for x in os.environ.get("FM_REFILL", "0").split(",")]
        packs = [int(x) for x in os.environ.get("FM_PACKED", "1").split(",")]
        for step, refill, packed in [(s_, r_, p_) for s_ in steps for r_ in (refills if s_ == 3 else [8])
                                     for p_ in (packs if s_ == 3 else [1])]:
            qr.qr_set_tuning("fm_step", step)
            qr.qr_set_tuning("fm_refill", refill)
            qr.qr_set_tuning("fm_packed", packed)
            work = torch.zeros(2, dtype=torch.uint64, device=dev)
            qr.qr_fm_count_work(fm, pats, None, L, out, m, work, st)
            torch.cuda.synchronize()
            h = int(out.to(torch.int64).sum())
            ref = h if ref is None else ref
            ms = t(lambda: qr.qr_fm_count(fm, pats, None, L, out, m, st), reps=3 if name == "c5" else 10)
            ok = int(out.to(torch.int64).sum()) == ref and h == ref
            steps_, lines = (int(x) for x in work.cpu())
            lps = lines / ms / 1e6
            print(json.dumps(dict(cfg=name, layout=lname, step=step, refill=refill, packed=packed, ms=round(ms, 4), gpat_s=round(m / ms / 1e6, 4),
                                  lines_per_pattern=lines / m, steps_per_pattern=steps_ / m, glines_s=round(lps, 3),
                                  frac_of_ceiling=round(lps / max(ceil.values()), 4), checksum_ok=ok)), flush=True)
        qr.qr_set_tuning("fm_step", 0)
        fm.free()
        torch.cuda.empty_cache()
    del txt, pats, out
    torch.cuda.empty_cache()
