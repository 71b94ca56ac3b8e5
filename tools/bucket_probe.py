"""Bucketed vs direct BiRank16 rank (bucket.cu) on one B200: configs[1] (2^34 bits, 10^9 queries)
and the 2^35-bit structure; parity of the two paths on the full batch (element by element on
the device), then Gq/s of each.  With --ncu only the bucketed path runs (launch list per pass).
Measurement only; the oracle parity is in tests/test_gpu_bucket.py.
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
ncu = "--ncu" in sys.argv


def t(fn, reps=5, warm=2):
    for _ in range(warm):
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


M = 1_000_000_000
q = torch.empty(M, dtype=torch.uint64, device=dev)
out = torch.empty_like(q)
ref = torch.empty_like(q)
for n in ([1 << 34] if ncu else [1 << 34, 1 << 35]):
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev)
    gen.bits_dev(1, n, 0.5, bits)
    h = qr.qr_birank_build(bits, n)
    del bits
    gen.queries_dev(1, n, M, q)
    if ncu:
        qr.qr_set_tuning("rank_bucket", 2)
        t(lambda: qr.qr_rank(h, q, None, out, M, st), reps=1, warm=1)
        break
    qr.qr_set_tuning("rank_bucket", 0)
    ms_d = t(lambda: qr.qr_rank(h, q, None, ref, M, st))
    qr.qr_set_tuning("rank_bucket", 2)
    ms_b = t(lambda: qr.qr_rank(h, q, None, out, M, st))
    same = bool(torch.equal(out.view(torch.int64), ref.view(torch.int64)))
    emit(n=n, m=M, direct_ms=ms_d, direct_gq_s=M / ms_d / 1e6, bucket_ms=ms_b, bucket_gq_s=M / ms_b / 1e6,
         identical=same)
    qr.qr_set_tuning("rank_bucket", 1)
    h.free()
