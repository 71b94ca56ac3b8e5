"""(Experiment tool; needs the rank_l2_pin_mb / persisting_l2_mb knobs of the commit that measured it, since removed.)
BiRank16 cluster rank kernel with an L2-pinned slice of the line array (evict_last for lines
below a threshold, evict_first above), with and without a persisting-L2 set-aside."""
import json, os, sys
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
M = 10**9
n = 1 << 34
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(2, n, 0.5, bits)
h = qr.qr_birank_build(bits, n); del bits
q = torch.empty(M, dtype=torch.uint64, device=dev); gen.queries_dev(2, n, M, q); out = torch.empty_like(q)
out0 = torch.empty_like(q)
qr.qr_rank(h, q, None, out0, M, st)
for persist in (0, 64, 96):
    try:
        qr.qr_set_tuning("persisting_l2_mb", persist)
    except Exception as e:
        print(json.dumps({"persist": persist, "error": str(e)})); continue
    for pin in (0, 32, 64, 80, 96, 112):
        qr.qr_set_tuning("rank_l2_pin_mb", pin)
        r = {"persist_mb": persist, "pin_mb": pin}
        r["gq_s"] = M / t(lambda: qr.qr_rank(h, q, None, out, M, st)) / 1e6
        torch.cuda.synchronize(); r["equal"] = bool(torch.equal(out, out0))
        print(json.dumps(r), flush=True)

qr.qr_set_tuning("persisting_l2_mb", 0)
