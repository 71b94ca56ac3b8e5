"""QuadFm count kernel sweep (lane-pair vs one lane per pattern, grid size) on configs 4 and 5."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for name, n, kind, m, L, seed in (("c4", 1 << 26, 0, 10**7, 32, 4), ("c5", 1 << 30, 1, 10**8, 100, 5)):
    txt = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev); gen.dna_dev(seed, n, kind, txt)
    fm = qr.qr_fm_build(txt, n, kmer_k=int(os.environ.get("KMER", "8")))
    pats = torch.empty(m * L, dtype=torch.uint8, device=dev); gen.patterns_dev(seed, 0 if kind == 0 else 1, m, L, txt, n, pats)
    out = torch.empty(m, dtype=torch.int32, device=dev)
    ref = None
    for pair in (1, 2):                     # here: fm_step flavour (1 = de-duplicating, 2 = lean)
        for bps in (64,):
            qr.qr_set_tuning("fm_step", pair); qr.qr_set_tuning("fm_blocks_per_sm", bps)
            ms = t(lambda: qr.qr_fm_count(fm, pats, None, L, out, m, st), reps=3 if name == "c5" else 10)
            h = int(out.view(torch.int32).to(torch.int64).sum())
            ref = h if ref is None else ref
            print(json.dumps(dict(cfg=name, kmer=fm.kmer_k, pair=pair, bps=bps, ms=ms, gpat_s=m / ms / 1e6, checksum_ok=(h == ref))), flush=True)
    fm.free(); del txt, pats, out; torch.cuda.empty_cache()
qr.qr_set_tuning("fm_step", 0); qr.qr_set_tuning("fm_blocks_per_sm", 64)
