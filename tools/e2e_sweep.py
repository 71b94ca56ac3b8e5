"""Staged host-pointer path sweep (chunk size x slots) for qr_rank with pinned host buffers."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n); del bits
me = 2 * 10**8
qd = torch.empty(me, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, me, qd)
qh = torch.empty(me, dtype=torch.uint64).pin_memory(); qh.copy_(qd.cpu())
oh = torch.empty(me, dtype=torch.uint64).pin_memory()
t0 = time.perf_counter(); x = qd.cpu(); h2d_ref = None
a = torch.empty(me, dtype=torch.uint64, device=dev)
torch.cuda.synchronize(); t0 = time.perf_counter(); a.copy_(qh, non_blocking=True); torch.cuda.synchronize()
h2d = 8 * me / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter(); oh.copy_(a, non_blocking=True); torch.cuda.synchronize()
d2h = 8 * me / (time.perf_counter() - t0) / 1e9
print(json.dumps(dict(plain_copy_h2d_gbs=h2d, plain_copy_d2h_gbs=d2h)), flush=True)
del a
for slots in (2, 3, 4):
    for chunk in (1 << 22, 1 << 23, 1 << 24, 1 << 25, 1 << 26):
        qr.qr_set_tuning("stage_slots", slots); qr.qr_set_tuning("stage_chunk", chunk)
        for _ in range(2):
            qr.qr_rank(h, qh, None, oh, me, st); st.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            qr.qr_rank(h, qh, None, oh, me, st); st.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / 3
        print(json.dumps(dict(slots=slots, chunk=chunk, ms=ms, gq_s=me / ms / 1e6, gbs_each_way=8 * me / ms / 1e6)), flush=True)
