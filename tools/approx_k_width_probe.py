"""Approximate counting (k = 1, 2, 3) on configs[3] vs the k-mer seed width of the index."""
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
n, m, L = 1 << 26, 10**6, 32
text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev); gen.dna_dev(4, n, 0, text)
pats = torch.empty(m * L, dtype=torch.uint8, device=dev); gen.patterns_dev(4, 0, m, L, text, n, pats)
out = torch.empty(m, dtype=torch.int32, device=dev)
for K in (6, 8, 10, 11, 12):
    fm = qr.qr_fm_build(text, n, kmer_k=K)
    for k, mk in ((1, m), (2, m), (3, m // 10)):
        ms = t(lambda: qr.qr_fm_count_approx(fm, pats, None, L, k, out, mk, st))
        print(json.dumps({"K": K, "k": k, "m": mk, "ms": ms, "gpat_s": mk / ms / 1e6,
                          "checksum": int(out[:mk].to(torch.int64).sum())}), flush=True)
    del fm
