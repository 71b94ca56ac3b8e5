"""L2-resident structures: which rank kernel shape is fastest (one lane per query vs lane pairs,
superblock words from L2 vs cluster shared memory, K)."""
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
M = 2 * 10**8
q = torch.empty(M, dtype=torch.uint64, device=dev); out = torch.empty_like(q); ref = torch.empty_like(q)
c = torch.empty(M, dtype=torch.uint8, device=dev)
CFG = [("pair_smem", 2, 1, 2, 4), ("pair_global", 0, 1, 2, 2), ("pair_global_k4", 0, 1, 4, 2),
       ("lane_global_k2", 0, 0, 2, 2), ("lane_global_k4", 0, 0, 4, 2), ("lane_global_k8", 0, 0, 8, 2)]
for sigma, lg in ((2, 26), (2, 28), (2, 30), (4, 26), (4, 28)):
    n = 1 << lg
    if sigma == 2:
        bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev); gen.bits_dev(7, n, 0.5, bits)
        h = qr.qr_birank_build(bits, n); del bits
        gen.queries_dev(8, n, M, q); cc = None
    else:
        text = torch.empty((n + 31) // 32, dtype=torch.uint64, device=dev); gen.dna_dev(9, n, 0, text)
        h = qr.qr_quadrank_build(text, n); del text
        gen.queries_dev(10, n, M, q, c); cc = c
    qr.qr_set_tuning("rank_smem", 0); qr.qr_set_tuning("rank_pair", 1); qr.qr_set_tuning("rank_k", 2)
    qr.qr_rank(h, q, cc, ref, M, st)
    r = {"sigma": sigma, "log2_n": lg}
    for name, smem, pair, k, sk in CFG:
        qr.qr_set_tuning("rank_smem", smem); qr.qr_set_tuning("rank_pair", pair); qr.qr_set_tuning("rank_k", k)
        qr.qr_set_tuning("rank_smem_k", 0)
        r[name] = round(M / t(lambda: qr.qr_rank(h, q, cc, out, M, st)) / 1e6, 2)
        torch.cuda.synchronize()
        if not torch.equal(out, ref): r[name + "_MISMATCH"] = True
    for bps in (8, 16, 32):
        qr.qr_set_tuning("rank_smem", 0); qr.qr_set_tuning("rank_pair", 0); qr.qr_set_tuning("rank_k", 4)
        qr.qr_set_tuning("rank_blocks_per_sm", bps)
        r[f"lane_global_k4_bps{bps}"] = round(M / t(lambda: qr.qr_rank(h, q, cc, out, M, st)) / 1e6, 2)
    qr.qr_set_tuning("rank_blocks_per_sm", 64)
    print(json.dumps(r), flush=True)
    h.free(); torch.cuda.empty_cache()
qr.qr_set_tuning("rank_smem", 1); qr.qr_set_tuning("rank_pair", 1); qr.qr_set_tuning("rank_k", 2)
