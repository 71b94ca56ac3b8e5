"""QuadFm count vs k-mer table width K (fast key path for K <= 16 when len >= 16) on configs[3],
configs[4] and the 150-bp reads (both strands); counts must not depend on K."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for name, n, kind, m, L, seed, pkind in (("c4", 1 << 26, 0, 10**7, 32, 4, 0), ("c5", 1 << 30, 1, 10**8, 100, 5, 1),
                                         ("reads150", 1 << 30, 1, 10**7, 150, 55, 2)):
    text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
    gen.dna_dev(seed if name != "reads150" else 5, n, kind, text)
    pats = torch.empty(m * L, dtype=torch.uint8, device=dev)
    gen.patterns_dev(seed, pkind, m, L, text, n, pats)
    ref = None
    for K in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["8", "12", "14"])]:
        t0 = time.perf_counter()
        fm = qr.qr_fm_build(text, n, kmer_k=K)
        bt = time.perf_counter() - t0
        out = torch.empty(m, dtype=torch.int32, device=dev)
        if name == "reads150":
            orc = torch.empty_like(out)
            ms = t(lambda: qr.qr_fm_count_both(fm, pats, None, L, out, orc, m, st))
            res = torch.cat([out, orc])
        else:
            ms = t(lambda: qr.qr_fm_count(fm, pats, None, L, out, m, st))
            res = out.clone()
        torch.cuda.synchronize()
        if ref is None: ref = res
        print(json.dumps({"cfg": name, "K": K, "ms": ms, "gpat_s": m / ms / 1e6, "build_s": round(bt, 3),
                          "equal_to_first": bool(torch.equal(res, ref))}), flush=True)
        del fm
        torch.cuda.empty_cache()
    del text, pats, ref
    torch.cuda.empty_cache()
