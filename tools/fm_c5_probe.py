"""QuadFm count on configs[3] / configs[4] at the library's defaults (one line per config)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
tag = sys.argv[1] if len(sys.argv) > 1 else ""
def t(fn, reps=5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for name, n, kind, m, L, seed in (("c4", 1 << 26, 0, 10**7, 32, 4), ("c5", 1 << 30, 1, 10**8, 100, 5)):
    text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
    gen.dna_dev(seed, n, kind, text)
    fm = qr.qr_fm_build(text, n)
    pats = torch.empty(m * L, dtype=torch.uint8, device=dev)
    gen.patterns_dev(seed, kind, m, L, text, n, pats)
    out = torch.empty(m, dtype=torch.int32, device=dev)
    for step in (0, 1, 2):
        qr.qr_set_tuning("fm_step", step)
        ms = t(lambda: qr.qr_fm_count(fm, pats, None, L, out, m, st))
        print(json.dumps({"tag": tag, "cfg": name, "step": step, "ms": ms, "gpat_s": m / ms / 1e6,
                          "checksum": int(out.to(torch.int64).sum())}), flush=True)
    qr.qr_set_tuning("fm_step", 0)
    del fm, text, pats, out
    torch.cuda.empty_cache()
