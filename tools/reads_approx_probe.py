"""The paper's reads (150 bp, 1% substitutions, either strand) on the configs[4] text: both
strands within k = 0..2 substitutions (qr_fm_count_approx_both), both BWT layouts."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=3):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
n, L = 1 << 30, 150
text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev); gen.dna_dev(5, n, 1, text)
for name, lay in (("quadrank16", qr.QR_LAYOUT_QUADRANK16), ("quadrank16x2", qr.QR_LAYOUT_QUADRANK16X2)):
    fm = qr.qr_fm_build(text, n, bwt_layout=lay, kmer_k=int(os.environ.get("QR_PROBE_K", "-1")))
    for k, m in ((0, 10**7), (1, 10**6), (2, 10**5)):
        pats = torch.empty(m * L, dtype=torch.uint8, device=dev); gen.patterns_dev(55, 2, m, L, text, n, pats)
        of = torch.empty(m, dtype=torch.int32, device=dev); orc = torch.empty_like(of)
        ms = t(lambda: qr.qr_fm_count_approx_both(fm, pats, None, L, k, of, orc, m, st))
        hit = float(((of > 0) | (orc > 0)).float().mean())
        print(json.dumps({"bwt": name, "k": k, "reads": m, "ms": ms, "reads_per_s": m / ms * 1e3,
                          "frac_reads_matching": hit}), flush=True)
    del fm
