"""Per-call cost of small qr_rank batches (host overhead + launch): 2000 back-to-back calls,
device pointers, wall clock and CUDA events."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
n = 1 << 20
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(1, n, 0.5, bits)
h = qr.qr_birank_build(bits, n)
for m in (1, 1000, 100000, 10**6, 4 * 10**6):
    q = torch.empty(m, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, m, q); out = torch.empty_like(q)
    for _ in range(50): qr.qr_rank(h, q, None, out, m, st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 2000
    t0 = time.perf_counter(); a.record(st)
    for _ in range(R): qr.qr_rank(h, q, None, out, m, st)
    t1 = time.perf_counter(); b.record(st); torch.cuda.synchronize()
    print(json.dumps({"m": m, "host_us_per_call": (t1 - t0) / R * 1e6, "gpu_us_per_call": a.elapsed_time(b) / R * 1e3}), flush=True)
