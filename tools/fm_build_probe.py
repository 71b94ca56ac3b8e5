"""QuadFm build time on configs[4] (2^30 block-repeat text) and the 3.1 Gbp text: wall time of
qr_fm_build (GPU suffix sort + BWT + QuadRank layout + k-mer table), per width.  Run under
`ncu --metrics gpu__time_duration.sum` with argv[1] = "once" for the per-kernel breakdown."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0")
once = len(sys.argv) > 1 and sys.argv[1] == "once"
sizes = ((1 << 30, 5, "c5"),) if once else ((1 << 26, 4, "c4"), (1 << 30, 5, "c5"), (3_100_000_000, 5, "3.1G"))
for n, seed, name in sizes:
    text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev)
    gen.dna_dev(seed, n, 0 if name == "c4" else 1, text)
    torch.cuda.synchronize()
    for k in ((12,) if once else (0, 12)):
        reps = 1 if once else 3
        ts = []
        for _ in range(reps + (0 if once else 1)):
            t0 = time.perf_counter()
            fm = qr.qr_fm_build(text, n, kmer_k=k)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            del fm
        print(json.dumps({"cfg": name, "n": n, "kmer_k": k, "build_s": ts, "best_s": min(ts[-reps:])}), flush=True)
    del text
    torch.cuda.empty_cache()
