"""Launch-configuration and gather-ceiling sweep for the rank kernels on one B200.

Prints one JSON line per measurement: kernel, structure size, K (queries per thread),
CTAs per SM, L2 fetch granularity, Gq/s.  Measurement only (no parity; tests do that).
"""
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


def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def emit(**kw):
    print(json.dumps(kw), flush=True)


def build_bi(n):
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev)
    gen.bits_dev(2, n, 0.5, bits)
    h = qr.qr_birank_build(bits, n)
    del bits
    return h


M = 400_000_000
q = torch.empty(M, dtype=torch.uint64, device=dev)
out = torch.empty_like(q)

# 1. launch grid for the headline structure
n = 1 << 34
h = build_bi(n)
gen.queries_dev(2, n, M, q)
for k in (1, 2, 4, 8):
    for bps in (2, 4, 8, 16, 32):
        qr.qr_set_tuning("rank_k", k)
        qr.qr_set_tuning("rank_blocks_per_sm", bps)
        ms = t(lambda: qr.qr_rank(h, q, None, out, M, st))
        g0 = t(lambda: qr.qr_gather_ceiling(h, q, out, 0, M, st))
        emit(kernel="bi_rank", n=n, K=k, bps=bps, gq_s=M / ms / 1e6, ceil0_gq_s=M / g0 / 1e6)
qr.qr_set_tuning("rank_k", 4)
qr.qr_set_tuning("rank_blocks_per_sm", 8)
# 2. L2 fetch granularity
for g in (32, 64, 128, 0):
    try:
        qr.qr_set_tuning("l2_fetch_granularity", g)
    except Exception as e:
        emit(l2_gran=g, error=str(e))
        continue
    ms = t(lambda: qr.qr_rank(h, q, None, out, M, st))
    g0 = t(lambda: qr.qr_gather_ceiling(h, q, out, 0, M, st))
    g1 = t(lambda: qr.qr_gather_ceiling(h, q, out, 1, M, st))
    emit(kernel="bi_rank", l2_gran=g, gq_s=M / ms / 1e6, ceil0_gq_s=M / g0 / 1e6, ceil1_gq_s=M / g1 / 1e6)
qr.qr_set_tuning("l2_fetch_granularity", 64)
# 3. sorted queries (line reuse through L2) and sequential lines (streaming)
qs, _ = torch.sort(q.view(torch.int64))
qs = qs.view(torch.uint64)
ms = t(lambda: qr.qr_rank(h, qs, None, out, M, st))
emit(kernel="bi_rank", order="sorted", gq_s=M / ms / 1e6)
L = n // 496 + 1
seq = (torch.arange(min(M, L), device=dev, dtype=torch.int64) * 496 + 300).view(torch.uint64)
ms = t(lambda: qr.qr_gather_ceiling(h, seq, out, 1, seq.numel(), st))
emit(kernel="gather_mode1", order="sequential_lines", lines=seq.numel(), gbs=seq.numel() * 80 / ms / 1e6)
h.free()
del qs, seq
torch.cuda.empty_cache()
# 4. structure size (HBM-resident random gather vs L2-resident)
for lg in (20, 26, 28, 30, 32, 34, 36):
    n = 1 << lg
    h = build_bi(n)
    gen.queries_dev(3, n, M, q)
    ms = t(lambda: qr.qr_rank(h, q, None, out, M, st))
    g0 = t(lambda: qr.qr_gather_ceiling(h, q, out, 0, M, st))
    g1 = t(lambda: qr.qr_gather_ceiling(h, q, out, 1, M, st))
    emit(kernel="bi_rank", n=n, line_bytes=h.line_bytes, gq_s=M / ms / 1e6, ceil0_gq_s=M / g0 / 1e6,
         ceil1_gq_s=M / g1 / 1e6)
    h.free()
    torch.cuda.empty_cache()
