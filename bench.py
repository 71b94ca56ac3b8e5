#!/usr/bin/env python
"""Benchmark of the hot path on B200 (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--rows all|headline]

Headline (`value`): BiRank16 rank queries/s on configs[1] (n = 2^34 bits, p = 0.5, 10^9 queries
per GPU, u64 out), whole job over N GPUs (weak scaling: each GPU keeps its 10^9 queries),
CUDA-event time on the launching stream, max over ranks.  `rows` adds every other §8(a) row
measured in the same run — p = 0.01, QuadRank rank / rank_all4 on configs[2], QuadFm count on
configs[3] and configs[4] (patterns strong-scaled over the N GPUs), configs[4]'s 8 x 10^9 rank
queries strong-scaled, the paper's 150-bp reads on both strands, approximate search, the layout
variants, latency mode and the small configs[0] — each with its own roofline (FM rows: lines/s
against the random-gather ceiling measured on the same BWT handle), clocks sampled during its
timed region, and an output checksum summed over the ranks (identical at every N).  Inputs are
created on the device from the seeded generators before the timed region; every timed input of
the HBM rows is far larger than the 126 MB L2 (no flush needed); the L2-resident FM rows are
L2-resident by design (configs[3]: an 18-22 MB BWT) and say so.

cpu_baseline: the oracle (oracle/, plain C, OpenMP over queries) timed on rank 0's host cores on
bounded samples of the same workloads after the GPU rows (at every N); its precompute (prefix
arrays, suffix array) runs in a background thread during the GPU rows and is not timed.

--impl reference: the CPU oracle timed on the host cores on a bounded sample of the headline
workload each step; rank 0 only.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rank Gqueries/s & HBM gather GB/s vs roofline; QuadFm patterns/s @1/2/4/8"
N2, M2 = 1 << 34, 10**9                 # configs[1]
N3, M3 = 1 << 32, 10**9                 # configs[2]
N4, M4, L4 = 1 << 26, 10**7, 32         # configs[3]
N5, M5, L5 = 1 << 30, 10**8, 100        # configs[4] (patterns)
R5 = 8 * 10**9                          # configs[4] rank queries, strong-scaled over the GPUs
N1, M1 = 1 << 20, 10**6                 # configs[0]
SEED = {1: 1, 2: 2, 3: 3, 4: 4, 5: 5}
# expected bytes of one BiRank query: sector 0 always, sector 1 when the
# query lies right of the anchor (data bits [240,496): 256/496 of uniform q) + 8 B q + 8 B out
BI_LINE_BYTES = 32 + 32 * 256 / 496
QD_LINE_BYTES = 32 + 32 * 128 / 224     # data chars [96,224) of 224 need sector 1
CEIL_Q = 1 << 26                        # queries of an FM row's gather-ceiling measurement


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms for the whole run; every timed
    region records its wall-clock window and gets the statistics of the samples inside it."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,temperature.gpu,"
              "temperature.memory,clocks.mem,serial")
    REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None
        self.samples = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        self.samples = []
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                sm, mx = float(p[2]), float(p[3])
            except ValueError:
                continue
            rs = {name for k, name in enumerate(self.REASONS) if p[6 + k].lower().startswith("active")}
            extra = []
            for k in (10, 11, 12):                  # GPU / HBM temperature, memory clock
                try:
                    extra.append(float(p[k]))
                except (ValueError, IndexError):
                    extra.append(None)
            self.samples.append((ts, sm, mx, rs, extra, p[13] if len(p) > 13 else None))
        os.unlink(self.path)

    def window(self, t0: float, t1: float, full: bool = False) -> dict:
        if self.proc is None or self.samples is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        s = [x for x in self.samples if t0 - 0.05 <= x[0] <= t1 + 0.05]
        if not s:                                   # a region shorter than the sampling period
            s = sorted(self.samples, key=lambda x: abs(x[0] - 0.5 * (t0 + t1)))[:1]
        med = lambda v: statistics.median(v) if v else None   # noqa: E731
        out = {"sm_mhz": med([x[1] for x in s]), "sm_max_mhz": s[-1][2] if s else None,
               "reasons": sorted(set().union(*[x[3] for x in s])) if s else [], "samples": len(s)}
        if full:
            out.update({"gpu_temp_c": med([x[4][0] for x in s if x[4][0] is not None]),
                        "hbm_temp_c": med([x[4][1] for x in s if x[4][1] is not None]),
                        "mem_mhz": med([x[4][2] for x in s if x[4][2] is not None]),
                        "gpu_serial": s[-1][5] if s else None})
        return out


class RowSkipped(Exception):
    pass


class Ctx:
    def __init__(self, args):
        import torch

        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.args = args
        self.dist = None
        ndev = max(1, torch.cuda.device_count())
        self.gpu = self.local % ndev        # one process per GPU; modulo only for the 1-GPU gloo smoke
        if self.world > 1:
            import torch.distributed as dist

            torch.cuda.set_device(self.gpu)
            if args.dist_backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.gpu))
            else:
                dist.init_process_group(args.dist_backend)
            self.dist = dist
        else:
            torch.cuda.set_device(0)
        self.dev = torch.device("cuda", self.gpu)
        self.stream = torch.cuda.current_stream()
        self.last_win = (0.0, 0.0)

    def _cd(self):                           # the device collectives run on (cpu for gloo)
        return self.dev if (self.dist and self.args.dist_backend == "nccl") else "cpu"

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self._cd())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, x: int) -> int:
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.int64, device=self._cd())
        self.dist.all_reduce(t)
        return int(t.item())

    def sum_u64_over_ranks(self, x: int) -> int:
        """sum mod 2^64 of one u64 per rank (multigpu.reduce_sum_u64)."""
        from paper_2602_04103_b200.multigpu import reduce_sum_u64

        return reduce_sum_u64(x, self.dist, self._cd())

    def gather_u64(self, x: int) -> list:
        from paper_2602_04103_b200.multigpu import gather_u64

        return gather_u64(x, self.dist, self._cd())

    def agree(self, ok: bool) -> bool:
        """True iff every rank is ok (one all_reduce MIN): a row that failed on one rank before its
        timed region (e.g. out of memory while building) is skipped by every rank, instead of
        leaving the others waiting in a collective."""
        if not self.dist:
            return ok
        t = self.torch.tensor([1 if ok else 0], dtype=self.torch.int64, device=self._cd())
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return bool(t.item())

    def timed(self, fn, steps: int, warmup: int) -> float:
        """ms per step: W warm-up calls, then EXACTLY K calls bracketed by barrier + synchronize,
        CUDA events on the launching stream, max over ranks.  The wall window is kept for clocks."""
        if self.dist and not self.agree(True):
            raise RowSkipped("another rank failed before this timed region")
        torch = self.torch
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        self.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record(self.stream)
        for i in range(steps):
            fn()
            ev[i + 1].record(self.stream)
        torch.cuda.synchronize()
        self.last_win = (t0, time.time())
        self.barrier()
        ms = ev[0].elapsed_time(ev[-1]) / steps
        # per-step times (median and minimum beside the mean), kept for the caller
        per = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(steps))
        self.last_step_ms = {"median": self.max_over_ranks(per[len(per) // 2]), "min": self.max_over_ranks(per[0])}
        return self.max_over_ranks(ms)

    def checksum(self, buf, count: int, word_bytes: int, index0: int) -> int:
        """qr_checksum of this rank's outputs (global indices index0..) on this rank."""
        import paper_2602_04103_b200 as qr

        acc = self.torch.zeros(1, dtype=self.torch.uint64, device=self.dev)
        qr.qr_checksum(buf, count, word_bytes, index0, acc, self.stream)
        self.torch.cuda.synchronize()
        return int(acc.view(self.torch.int64).item()) & (2**64 - 1)


def shard(total, world, rank):
    """contiguous shard of a global index range (paper_2602_04103_b200.multigpu.shard), imported
    lazily: the product package loads libqrank.so on import, which the reference arm must not."""
    from paper_2602_04103_b200.multigpu import shard as _shard

    return _shard(total, world, rank)


def hexs(x: int) -> str:
    return f"{x & (2**64 - 1):016x}"


# ------------------------------------------------------------------ rows
def bench_birank(ctx, p: float, steps, warmup, with_ceiling: bool, e2e=False):
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    seed_bits = SEED[2] if p == 0.5 else 22
    if ctx.dist and ctx.args.replicate == "broadcast":
        # rank 0 builds; the layout is broadcast to every rank (NCCL over NVLink) and imported
        from paper_2602_04103_b200.multigpu import broadcast_index

        h0 = None
        if ctx.rank == 0:
            bits = torch.empty((N2 + 63) // 64, dtype=torch.uint64, device=ctx.dev)
            gen.bits_dev(seed_bits, N2, p, bits)
            h0 = qr.qr_birank_build(bits, N2, device=ctx.gpu)
            del bits
        h = broadcast_index(h0, N2, qr.QR_LAYOUT_BIRANK16, ctx.dist, ctx.dev)
    else:
        bits = torch.empty((N2 + 63) // 64, dtype=torch.uint64, device=ctx.dev)
        gen.bits_dev(seed_bits, N2, p, bits)
        h = qr.qr_birank_build(bits, N2, device=ctx.gpu)
        del bits
    m = M2                                         # per GPU (weak scaling)
    i0 = ctx.rank * m
    q = torch.empty(m, dtype=torch.uint64, device=ctx.dev)
    gen.queries_dev(SEED[2], N2, m, q, i0=i0)
    out = torch.empty_like(q)
    torch.cuda.synchronize()
    ms = ctx.timed(lambda: qr.qr_rank(h, q, None, out, m, ctx.stream), steps, warmup)
    res = {"ms": ms, "m_per_gpu": m, "gq_s": ctx.world * m / ms / 1e6, "launches": steps, "_win": ctx.last_win,
           "step_ms": dict(ctx.last_step_ms)}
    res["smem_cache_cta_bytes"] = qr.qr_super_cache_bytes(h)
    # output checksums (qr_checksum over global query indices): this rank's shard, the sum over
    # the ranks, and a cross-GPU check — rank r recomputes shard (r+1) mod N untimed and must get
    # the checksum that rank reported.  Shard 0 is the same 10^9 queries at every N.
    own = ctx.checksum(out, m, 8, i0)
    allc = ctx.gather_u64(own)
    nxt = (ctx.rank + 1) % ctx.world
    gen.queries_dev(SEED[2], N2, m, q, i0=nxt * m)
    qr.qr_rank(h, q, None, out, m, ctx.stream)
    cross_ok = ctx.checksum(out, m, 8, nxt * m) == allc[nxt]
    cross_ok = ctx.sum_over_ranks(int(cross_ok)) == ctx.world
    gen.queries_dev(SEED[2], N2, m, q, i0=i0)
    res["checksum"] = {"shard0": hexs(allc[0]), "all_ranks_sum": hexs(sum(allc)), "cross_gpu_recompute_ok": cross_ok,
                       "scheme": "sum_i mix(global query index i, rank value) mod 2^64 (qr_checksum)"}
    if with_ceiling:
        # modes 0-2: the global-memory lane-pair kernel's loads (lines only, full lines, lines +
        # superblock word); mode 3: the cluster kernel's own launch shape and line loads, no s
        for mode in ((0, 1, 2, 3) if res["smem_cache_cta_bytes"] else (0, 1, 2)):
            cms = ctx.timed(lambda: qr.qr_gather_ceiling(h, q, out, mode, m, ctx.stream), steps, warmup)
            res[f"ceiling_mode{mode}"] = {"ms": cms, "gq_s": ctx.world * m / cms / 1e6}
    if e2e:
        # the full per-GPU batch from pinned host memory at N = 1; at N > 1 each rank stages
        # M2 / N queries so that the box pins ~16 GB in total, not 16 GB per GPU
        me = M2 if ctx.world == 1 else max(10**8, M2 // ctx.world)
        from paper_2602_04103_b200.multigpu import on_gpu_local_cpus

        with on_gpu_local_cpus(ctx.dev.index or 0):     # pinned pages on the GPU's NUMA node
            qh = torch.empty(me, dtype=torch.uint64).pin_memory()
            oh = torch.empty(me, dtype=torch.uint64).pin_memory()
        qh.copy_(q[:me])

        def call():
            qr.qr_rank(h, qh, None, oh, me, ctx.stream)
            ctx.stream.synchronize()
            _ = int(oh[-1])                        # the D2H result is read by the host
        for _ in range(2):
            call()
        torch.cuda.synchronize()
        ctx.barrier()
        t0w = time.time()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        k = max(3, steps)                          # ~0.17 s per step: K steps keep one host hiccup from dominating
        step_wall = []
        for _ in range(k):
            ts = time.perf_counter()
            call()
            step_wall.append((time.perf_counter() - ts) * 1e3)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3 / k
        ems = ctx.max_over_ranks(max(e0.elapsed_time(e1) / k, wall))
        res["e2e"] = {"value": round(ctx.world * me / ems / 1e6, 4), "unit": "Gqueries/s",
                      "h2d_bytes_per_step": 8 * me, "d2h_bytes_per_step": 8 * me, "queries_per_step": me,
                      "ms_per_step": round(ems, 3), "steps": k,
                      "ms_per_step_median": round(statistics.median(step_wall), 3),
                      "ms_per_step_max": round(max(step_wall), 3), "_win": (t0w, time.time())}
        del qh, oh
    del q, out
    h.free()
    torch.cuda.empty_cache()
    return res


def bench_birank_size(ctx, log2n, steps, warmup):
    """BiRank16 rank at the paper's own bit-vector size (4 GiB = 2^35 bits): the 4/8-CTA
    cluster superblock table path, 10^9 uniform queries per GPU."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    n = 1 << log2n
    bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=ctx.dev)
    gen.bits_dev(SEED[2], n, 0.5, bits)
    h = qr.qr_birank_build(bits, n, device=ctx.gpu)
    del bits
    m = M2
    q = torch.empty(m, dtype=torch.uint64, device=ctx.dev)
    gen.queries_dev(SEED[2], n, m, q, i0=ctx.rank * m)
    out = torch.empty_like(q)
    ms = ctx.timed(lambda: qr.qr_rank(h, q, None, out, m, ctx.stream), steps, warmup)
    h.free()
    del q, out
    torch.cuda.empty_cache()
    return {"ms": ms, "gq_s": ctx.world * m / ms / 1e6, "n_bits": n, "_win": ctx.last_win}


def rank_roofline(gq_s_per_gpu: float, bytes_per_q: float, peak: float) -> dict:
    a = gq_s_per_gpu * bytes_per_q
    return {"bound": "hbm", "achieved_gbs_per_gpu": round(a, 1), "peak": peak, "unit": "GB/s",
            "frac": round(a / peak, 4), "alg_bytes_per_query": round(bytes_per_q, 3)}


def bench_quadrank(ctx, steps, warmup, peak):
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    text = torch.empty((N3 + 31) // 32, dtype=torch.uint64, device=ctx.dev)
    gen.dna_dev(SEED[3], N3, 0, text)
    h = qr.qr_quadrank_build(text, N3, device=ctx.gpu)
    del text
    m = M3
    i0 = ctx.rank * m
    q = torch.empty(m, dtype=torch.uint64, device=ctx.dev)
    c = torch.empty(m, dtype=torch.uint8, device=ctx.dev)
    gen.queries_dev(SEED[3], N3, m, q, c, i0=i0)
    out = torch.empty_like(q)
    ms = ctx.timed(lambda: qr.qr_rank(h, q, c, out, m, ctx.stream), steps, warmup)
    w_rank = ctx.last_win
    cks = ctx.sum_u64_over_ranks(ctx.checksum(out, m, 8, i0))
    cms = ctx.timed(lambda: qr.qr_gather_ceiling(h, q, out, 0, m, ctx.stream), steps, warmup)
    del out
    out4 = torch.empty((m, 4), dtype=torch.uint64, device=ctx.dev)
    ms4 = ctx.timed(lambda: qr.qr_rank_all4(h, q, out4, m, ctx.stream), steps, warmup)
    w4 = ctx.last_win
    cks4 = ctx.sum_u64_over_ranks(ctx.checksum(out4, 4 * m, 8, 4 * i0))
    # rank_4's own ceiling: the same loads with its 32-B output stream (qr_gather_ceiling mode 4)
    cms4 = ctx.timed(lambda: qr.qr_gather_ceiling(h, q, out4, 4, m, ctx.stream), steps, warmup)
    del q, c, out4
    h.free()
    torch.cuda.empty_cache()
    g, g4 = m / ms / 1e6, m / ms4 / 1e6
    return {"rank": {"ms": ms, "gq_s": ctx.world * g, "_win": w_rank, "checksum": hexs(cks),
                     "roofline": dict(rank_roofline(g, QD_LINE_BYTES + 17, peak),
                                      frac_of_gather_ceiling=round(cms / ms, 4))},
            "ceiling_mode0": {"ms": cms, "gq_s": ctx.world * m / cms / 1e6},
            "rank_all4": {"ms": ms4, "gq_s": ctx.world * g4, "_win": w4, "checksum": hexs(cks4),
                          "roofline": dict(rank_roofline(g4, QD_LINE_BYTES + 40, peak),
                                           frac_of_gather_ceiling=round(cms4 / ms4, 4))},
            "ceiling_rank4_shape": {"ms": cms4, "gq_s": ctx.world * m / cms4 / 1e6}}


def fm_ceiling(ctx, fm, steps, warmup, seed):
    """Random-gather ceiling of a BWT handle (qr_gather_ceiling modes 0 and 1 on CEIL_Q uniform
    rows in [0, N]): G lines/s the memory system serves for this structure, per GPU."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    q = torch.empty(CEIL_Q, dtype=torch.uint64, device=ctx.dev)
    gen.queries_dev(seed + 100, fm.n + 1, CEIL_Q, q, i0=ctx.rank * CEIL_Q)
    o = torch.empty_like(q)
    modes = {}
    for mode in (0, 1):
        ms = ctx.timed(lambda: qr.qr_gather_ceiling(fm.bwt, q, o, mode, CEIL_Q, ctx.stream), steps, warmup)
        modes[mode] = CEIL_Q / ms / 1e6
    del q, o
    return max(modes.values()), modes


def bench_fm(ctx, n, kind, m_total, length, seed, steps, warmup, bwt_layout=None, rank_queries=0, strands=1,
             kmax=0, ptype=None):
    """QuadFm count (exact, one or both strands, or <= kmax substitutions) over the seeded text:
    patterns strong-scaled over the ranks, the work counted by qr_fm_count_work_ex (untimed), the
    BWT's gather ceiling measured on the same handle, an output checksum summed over the ranks."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=ctx.dev)
    gen.dna_dev(seed if ptype != 2 else 5, n, kind, text)
    t0 = time.perf_counter()
    fm = qr.qr_fm_build(text, n, device=ctx.gpu, bwt_layout=bwt_layout)
    build_s = time.perf_counter() - t0
    i0, m = shard(m_total, ctx.world, ctx.rank)
    pk = ptype if ptype is not None else (0 if kind == 0 else 1)
    pats = torch.empty(max(1, m * length), dtype=torch.uint8, device=ctx.dev)
    gen.patterns_dev(seed, pk, m, length, text, n, pats, i0=i0)
    out = torch.empty(m, dtype=torch.int32, device=ctx.dev)
    orc = torch.empty(m, dtype=torch.int32, device=ctx.dev) if strands == 2 else None
    work = torch.zeros(2, dtype=torch.uint64, device=ctx.dev)
    qr.qr_fm_count_work_ex(fm, pats, None, length, kmax, out, orc, m, work, ctx.stream)
    torch.cuda.synchronize()
    steps_done, lines = (int(x) for x in work.cpu())
    if kmax == 0 and strands == 1:
        call = lambda: qr.qr_fm_count(fm, pats, None, length, out, m, ctx.stream)   # noqa: E731
    elif kmax == 0:
        call = lambda: qr.qr_fm_count_both(fm, pats, None, length, out, orc, m, ctx.stream)   # noqa: E731
    elif strands == 1:
        call = lambda: qr.qr_fm_count_approx(fm, pats, None, length, kmax, out, m, ctx.stream)   # noqa: E731
    else:
        call = lambda: qr.qr_fm_count_approx_both(fm, pats, None, length, kmax, out, orc, m, ctx.stream)   # noqa: E731
    ms = ctx.timed(call, steps, warmup)
    win = ctx.last_win
    cks = ctx.checksum(out, m, 4, i0)
    if orc is not None:
        cks = (cks + ctx.checksum(orc, m, 4, m_total + i0)) & (2**64 - 1)
    cks = ctx.sum_u64_over_ranks(cks)
    hits = (out > 0) | (orc > 0) if orc is not None else (out > 0)
    hit = ctx.sum_over_ranks(int(hits.sum()))
    ceil, modes = fm_ceiling(ctx, fm, steps, warmup, seed)
    l2_res = fm.bwt.line_bytes <= 126 * 2**20 // 2
    steps_all, lines_all = ctx.sum_over_ranks(steps_done), ctx.sum_over_ranks(lines)
    # FM roofline: lines gathered per second per GPU ÷ the ceiling's lines/s on the
    # same BWT handle (the slowest rank's time, the whole job's lines)
    gl = lines_all / ctx.world / ms / 1e6
    res = {"ms": ms, "patterns_per_s": m_total / ms * 1e3, "searches_per_s": strands * m_total / ms * 1e3,
           "build_s": round(build_s, 3), "kmer_k": fm.kmer_k, "text_len": n, "patterns": m_total, "pattern_len": length,
           "strands": strands, "max_mismatches": kmax,
           "work_per_pattern": {"rank_pairs": steps_all / m_total, "lines": lines_all / m_total},
           "lines_per_s": lines_all / ms * 1e3,
           "alg_gbs": (lines_all * 64 + m_total * (length + 4 * strands)) / ms / 1e6,
           "frac_patterns_with_hits": hit / m_total, "checksum": hexs(cks), "_win": win,
           "bwt_bytes": fm.bwt.line_bytes, "bwt_residency": "L2 (fits in half of the 126 MB L2)" if l2_res else "HBM",
           "roofline": {"bound": "l2-random-gather" if l2_res else "hbm-random-gather", "unit": "G lines/s per GPU",
                        "achieved": round(gl, 3), "ceiling": round(ceil, 3), "frac": round(gl / ceil, 4),
                        "ceiling_modes": {str(k): round(v, 3) for k, v in modes.items()},
                        "ceiling_kind": "qr_gather_ceiling (best of modes 0/1) on this BWT handle, uniform rows in [0, N]"}}
    del pats, out, orc
    if rank_queries:
        res["rank_8e9_strong"] = bench_rank_on_bwt(ctx, fm, n, seed, rank_queries, steps, warmup)
    fm.free()
    del text
    torch.cuda.empty_cache()
    return res


def bench_rank_on_bwt(ctx, fm, n, seed, total, steps, warmup):
    """configs[4]'s rank queries (q, c) over the BWT's QuadRank16 layout, strong-scaled: this rank
    holds its total/N queries in HBM and ranks them in launches of <= 10^9 per step."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    i0, m = shard(total, ctx.world, ctx.rank)
    q = torch.empty(m, dtype=torch.uint64, device=ctx.dev)
    c = torch.empty(m, dtype=torch.uint8, device=ctx.dev)
    gen.queries_dev(seed, n + 1, m, q, c, i0=i0)
    chunk = min(m, 10**9)
    o = torch.empty(chunk, dtype=torch.uint64, device=ctx.dev)
    parts = [(a, min(m, a + chunk)) for a in range(0, m, chunk)]

    def call():
        for a, b in parts:
            qr.qr_rank(fm.bwt, q[a:b], c[a:b], o, b - a, ctx.stream)
    ms = ctx.timed(call, max(2, steps // 2), warmup)
    win = ctx.last_win
    cks = 0
    for a, b in parts:
        qr.qr_rank(fm.bwt, q[a:b], c[a:b], o, b - a, ctx.stream)
        cks += ctx.checksum(o, b - a, 8, i0 + a)
    cks = ctx.sum_u64_over_ranks(cks)
    del q, c, o
    torch.cuda.empty_cache()
    return {"ms": ms, "gq_s": total / ms / 1e6, "queries_total": total, "queries_per_gpu": m,
            "launches_per_step": len(parts), "scaling": "strong", "checksum": hexs(cks), "_win": win}


def bench_variants(ctx, steps, warmup):
    """The paper's evaluated layout variants (NEXT §8(f)4) on the configs[1] / configs[2] workloads."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    res = {}
    bits = torch.empty((N2 + 63) // 64, dtype=torch.uint64, device=ctx.dev)
    gen.bits_dev(SEED[2], N2, 0.5, bits)
    q = torch.empty(M2, dtype=torch.uint64, device=ctx.dev)
    gen.queries_dev(SEED[2], N2, M2, q, i0=ctx.rank * M2)
    out = torch.empty_like(q)
    for key, layout in (("c2_birank64x2", qr.QR_LAYOUT_BIRANK64X2), ("c2_birank16x2", qr.QR_LAYOUT_BIRANK16X2),
                        ("c2_birank32x2", qr.QR_LAYOUT_BIRANK32X2)):
        h = qr.qr_build(bits, N2, layout, device=ctx.gpu)
        ms = ctx.timed(lambda: qr.qr_rank(h, q, None, out, M2, ctx.stream), steps, warmup)
        res[key] = {"ms": ms, "gq_s": ctx.world * M2 / ms / 1e6, "bytes": h.line_bytes + h.super_bytes,
                    "overhead": (h.line_bytes + h.super_bytes) / (N2 / 8) - 1, "_win": ctx.last_win}
        h.free()
    del bits
    text = torch.empty((N3 + 31) // 32, dtype=torch.uint64, device=ctx.dev)
    gen.dna_dev(SEED[3], N3, 0, text)
    c = torch.empty(M3, dtype=torch.uint8, device=ctx.dev)
    gen.queries_dev(SEED[3], N3, M3, q, c, i0=ctx.rank * M3)
    o4 = torch.empty((M3, 4), dtype=torch.uint64, device=ctx.dev)
    for key, layout in (("c3_quadrank64", qr.QR_LAYOUT_QUADRANK64), ("c3_quadrank16x2", qr.QR_LAYOUT_QUADRANK16X2)):
        h = qr.qr_build(text, N3, layout, device=ctx.gpu)
        ms = ctx.timed(lambda: qr.qr_rank(h, q, c, out, M3, ctx.stream), steps, warmup)
        w = ctx.last_win
        ms4 = ctx.timed(lambda: qr.qr_rank_all4(h, q, o4, M3, ctx.stream), steps, warmup)
        res[key] = {"rank": {"ms": ms, "gq_s": ctx.world * M3 / ms / 1e6, "_win": w},
                    "rank_all4": {"ms": ms4, "gq_s": ctx.world * M3 / ms4 / 1e6, "_win": ctx.last_win},
                    "bytes": h.line_bytes + h.super_bytes, "overhead": (h.line_bytes + h.super_bytes) / (N3 / 4) - 1}
        h.free()
    del text, q, c, o4, out
    torch.cuda.empty_cache()
    return res


def bench_latency(ctx, steps, warmup):
    """Dependent-chain ("latency") mode vs the independent-query ("loop") mode on configs[1]
    (the paper reports ~80 ns per dependent query on DDR4)."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    bits = torch.empty((N2 + 63) // 64, dtype=torch.uint64, device=ctx.dev)
    gen.bits_dev(SEED[2], N2, 0.5, bits)
    res = {}
    for name, layout in (("birank16", qr.QR_LAYOUT_BIRANK16), ("birank64x2", qr.QR_LAYOUT_BIRANK64X2)):
        h = qr.qr_build(bits, N2, layout, device=ctx.gpu)
        L, chains = 2000, 148                          # one chain per SM: pure latency
        m = L * chains
        q = torch.empty(m, dtype=torch.uint64, device=ctx.dev)
        gen.queries_dev(SEED[2], N2, m, q)
        out = torch.empty_like(q)
        ms = ctx.timed(lambda: qr.qr_rank_chain(h, q, None, out, L, m, ctx.stream), max(2, steps // 2), warmup)
        w = ctx.last_win
        L2, chains2 = 200, 148 * 2048                  # many chains: latency-bound throughput
        m2 = L2 * chains2
        q2 = torch.empty(m2, dtype=torch.uint64, device=ctx.dev)
        gen.queries_dev(SEED[2] + 1, N2, m2, q2)
        out2 = torch.empty_like(q2)
        ms2 = ctx.timed(lambda: qr.qr_rank_chain(h, q2, None, out2, L2, m2, ctx.stream), max(2, steps // 2), warmup)
        res[name] = {"ns_per_dependent_query": ms * 1e6 / L, "chains": chains, "chain_len": L,
                     "many_chains_gq_s": m2 / ms2 / 1e6, "many_chains": chains2, "_win": (w[0], ctx.last_win[1])}
        h.free()
        del q, out, q2, out2
    del bits
    torch.cuda.empty_cache()
    return res


def bench_small(ctx, steps, warmup):
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    bits = torch.empty((N1 + 63) // 64, dtype=torch.uint64, device=ctx.dev)
    gen.bits_dev(SEED[1], N1, 0.5, bits)
    h = qr.qr_birank_build(bits, N1, device=ctx.gpu)
    q = torch.empty(M1, dtype=torch.uint64, device=ctx.dev)
    gen.queries_dev(SEED[1], N1, M1, q, i0=ctx.rank * M1)
    out = torch.empty_like(q)
    ms = ctx.timed(lambda: qr.qr_rank(h, q, None, out, M1, ctx.stream), steps * 10, warmup)
    h.free()
    return {"ms": ms, "gq_s": ctx.world * M1 / ms / 1e6, "_win": ctx.last_win,
            "note": "configs[0]: 135 KB structure, launch-dominated; not roofline-graded (SURVEY §8(d))"}


# ------------------------------------------------------------------ CPU oracle
class OraclePrep:
    """The oracles' precompute for the cpu_baseline rows (host-regenerated inputs, prefix arrays,
    the FM suffix array), run in a background thread while the GPU rows are timed (ctypes
    releases the GIL).  Timed afterwards on bounded samples; the precompute is reported, untimed."""

    def __init__(self, fm: bool = True):
        self.res = {}
        self.err = {}
        self.t = threading.Thread(target=self.run, args=(fm,), daemon=True)

    def start(self):
        self.t.start()
        return self

    def run(self, fm):
        import gen
        import oracle

        jobs = [("c2", lambda: oracle.BitsOracle(gen.bits(SEED[2], N2, 0.5), N2)),
                ("c3", lambda: oracle.DnaOracle(gen.dna(SEED[3], N3, 0), N3))]
        if fm:
            jobs.append(("c4", lambda: oracle.FmOracle(gen.unpack_dna(gen.dna(SEED[4], N4, 0), N4))))
        for key, fn in jobs:
            t0 = time.perf_counter()
            try:
                self.res[key] = (fn(), time.perf_counter() - t0)
            except Exception as e:                 # e.g. host memory
                self.err[key] = str(e)[:200]

    def get(self, key):
        self.t.join()
        return self.res.get(key, (None, None))


def _time_oracle(fn, target_s: float) -> tuple[float, int]:
    t0 = time.perf_counter()
    reps = 0
    while True:
        fn()
        reps += 1
        if time.perf_counter() - t0 > target_s:
            break
    return time.perf_counter() - t0, reps


def host_info() -> dict:
    """CPU model, logical CPUs and RAM of the host the oracle runs on."""
    info = {"nproc": os.cpu_count(), "cpus_allowed": len(os.sched_getaffinity(0))}
    try:
        with open("/proc/cpuinfo") as f:
            info["cpu_model"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    try:
        with open("/proc/meminfo") as f:
            info["ram_gb"] = round(int(next(l.split()[1] for l in f if l.startswith("MemTotal"))) / 2**20, 1)
    except (OSError, StopIteration):
        pass
    return info


def cpu_baselines(prep: OraclePrep, target_s: float = 10.0) -> dict:
    import numpy as np

    import gen
    import oracle

    oracle.set_threads(len(os.sched_getaffinity(0)))   # torchrun sets OMP_NUM_THREADS=1 per rank
    cores = oracle.threads()
    out = {"host": host_info()}
    ora, prep_s = prep.get("c2")
    if ora is not None:
        q = gen.queries(SEED[2], N2, 1 << 27)
        dt, reps = _time_oracle(lambda: ora.rank(q), target_s)
        out["c2_rank"] = {"value": round(reps * q.size / dt / 1e9, 6), "unit": "Gqueries/s", "cores": cores,
                          "kind": "oracle",
                          "sample": f"{q.size} queries of the configs[1] stream x {reps} passes ({dt:.1f}s of CPU work); "
                                    f"host-regenerated text 2^34 bits, plain prefix-array precompute {prep_s:.1f}s untimed"}
    ora, prep_s = prep.get("c3")
    if ora is not None:
        q, c = gen.queries(SEED[3], N3, 1 << 24, with_c=True)
        dt, reps = _time_oracle(lambda: ora.rank(q, c), target_s / 2)
        out["c3_rank"] = {"value": round(reps * q.size / dt / 1e9, 6), "unit": "Gqueries/s", "cores": cores,
                          "kind": "oracle", "sample": f"{q.size} (q, c) of the configs[2] stream x {reps} passes "
                                                      f"({dt:.1f}s); checkpoint precompute {prep_s:.1f}s untimed"}
        dt, reps = _time_oracle(lambda: ora.rank_all4(q), target_s / 2)
        out["c3_rank_all4"] = {"value": round(reps * q.size / dt / 1e9, 6), "unit": "Gqueries/s", "cores": cores,
                               "kind": "oracle", "sample": f"{q.size} q of the configs[2] stream x {reps} passes "
                                                           f"({dt:.1f}s); four rank calls per q"}
    ora, prep_s = prep.get("c4")
    if ora is not None:
        m = 2 * 10**6
        pats = gen.patterns(SEED[4], 0, m, L4, gen.dna(SEED[4], N4, 0), N4)
        offs, lens = np.arange(m, dtype=np.uint64) * L4, np.full(m, L4, np.uint32)
        dt, reps = _time_oracle(lambda: ora.count(pats, offs, lens), target_s / 2)
        out["c4_fm"] = {"value": round(reps * m / dt / 1e6, 4), "unit": "M patterns/s", "cores": cores,
                        "kind": "oracle",
                        "sample": f"{m} of the configs[3] patterns x {reps} passes ({dt:.1f}s); backward search over "
                                  f"the oracle's plain BWT, its suffix array precompute {prep_s:.1f}s untimed"}
    if prep.err:
        out["errors"] = prep.err
    return out


def cpu_oracle_rank(per_step_q: int):
    import gen
    import oracle

    t0 = time.perf_counter()
    ora = oracle.BitsOracle(gen.bits(SEED[2], N2, 0.5), N2)
    return ora, gen.queries(SEED[2], N2, per_step_q), time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the oracle timed on the host, same metric / config / unit."""
    import oracle

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    oracle.set_threads(len(os.sched_getaffinity(0)))   # torchrun sets OMP_NUM_THREADS=1 per rank
    ora, q, prep = cpu_oracle_rank(per_step_q=1 << 24)
    for _ in range(args.warmup):
        ora.rank(q)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ora.rank(q)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    v = q.size / ms / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "Gqueries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(args.gpus),
            "cpu_baseline": {"value": round(v, 6), "unit": "Gqueries/s", "cores": oracle.threads(), "kind": "oracle",
                             "sample": f"{q.size} of the configs[1] queries per step (host-regenerated), text 2^34 bits; "
                                       f"prefix-array precompute {prep:.1f}s untimed"},
            "e2e": {"value": round(v, 6), "unit": "Gqueries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_host": host_info(), "repo_so_loaded": repo_so_loaded()}
    print(json.dumps(line), flush=True)


def repo_so_loaded():
    """The repo's own shared libraries mapped into this process (the reference arm must show only
    oracle/ and gen/, never the product's libqrank.so)."""
    try:
        with open("/proc/self/maps") as f:
            paths = {l.split()[-1] for l in f if l.rstrip().endswith(".so") and ROOT in l}
        return sorted(os.path.relpath(p, ROOT) for p in paths)
    except OSError:
        return None


def workload_config(n_gpus):
    return {"workload": "configs[1]: BiRank16 rank, n=2^34 bits iid Bernoulli(0.5), 10^9 uniform q in [0,n] per GPU, "
                        "u64 out", "n_bits": N2, "queries_per_gpu": M2, "global_queries": M2 * n_gpus,
            "parallelism": f"replicate structure, shard queries x{n_gpus}",
            "l2": "no flush: timed inputs (2.2 GB lines, 8 GB queries) >> 126 MB L2"}


def traffic_record(alg_bytes_launch: float):
    """DRAM bytes per launch of the headline kernel from the committed ncu --set full capture,
    with its provenance (profiles/traffic.json, written by tools/ncu_traffic.py from that capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
    except Exception:
        return None, None
    t = tj.get("k_bi_rank_bytes_per_launch")
    if not t:
        return None, None
    src = {k: tj.get(k) for k in ("source", "kernel", "gpu_serial", "captured", "lib", "read_bytes", "write_bytes")}
    src["over_fetch"] = round(t / alg_bytes_launch, 4)
    src["note"] = ("ncu capture of this build's headline kernel (cold-cache, serialised replay); "
                   "over_fetch = traffic / algorithmic bytes: each query fills a whole 64-B line (.L2::64B)")
    return t, src


def finalize(obj, clocks: Clocks):
    """Replace every '_win' (wall window of a timed region) by the clocks sampled inside it."""
    if isinstance(obj, dict):
        out = {}
        for k, v in obj.items():
            if k == "_win":
                out["clocks"] = clocks.window(*v)
            else:
                out[k] = finalize(v, clocks)
        return out
    if isinstance(obj, list):
        return [finalize(v, clocks) for v in obj]
    return obj


def safe(ctx, fn):
    """A row that fails (e.g. out of memory on a smaller GPU) is reported, not fatal; under
    torchrun the failing rank tells the others at their next timed region (Ctx.agree)."""
    import torch

    try:
        torch.cuda.empty_cache()
        return fn()
    except RowSkipped as e:
        torch.cuda.empty_cache()
        return {"skipped": str(e)}
    except Exception as e:
        torch.cuda.empty_cache()
        if ctx.dist:
            ctx.agree(False)
        return {"skipped": f"{type(e).__name__}: {str(e)[:200]}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", default="all", choices=["all", "headline"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--only", default="", help="comma-separated row names (development runs; default: every row)")
    ap.add_argument("--replicate", default="build", choices=["build", "broadcast"],
                    help="multi-GPU: every rank builds from the seeded text, or rank 0 builds and broadcasts")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo only to smoke-test the multi-rank path on one GPU)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import paper_2602_04103_b200 as qr

    ctx = Ctx(args)
    for kv in filter(None, os.environ.get("QR_TUNING", "").split(",")):   # development runs only
        k, v = kv.split("=")
        qr.qr_set_tuning(k, int(v))
    K, W = args.steps, max(3, args.warmup)
    peak, peak_src = peaks()
    clocks = Clocks(ctx.gpu)
    clocks.start()
    prep = OraclePrep(fm=args.rows == "all").start() if (ctx.rank == 0 and not args.no_cpu) else None
    wall0 = time.perf_counter()
    c2 = bench_birank(ctx, 0.5, K, W, with_ceiling=True, e2e=True)
    rows = {}
    if args.rows == "all":
        X2 = qr.QR_LAYOUT_QUADRANK16X2
        spec = [
            ("c2_p0.01", lambda: bench_birank(ctx, 0.01, K, W, with_ceiling=False)),
            ("birank16_2^35_paper_size", lambda: bench_birank_size(ctx, 35, K, W)),
            ("c3_quadrank", lambda: bench_quadrank(ctx, K, W, peak)),
            ("c4_quadfm", lambda: bench_fm(ctx, N4, 0, M4, L4, SEED[4], K, W)),
            ("c4_quadfm_bwt16x2", lambda: bench_fm(ctx, N4, 0, M4, L4, SEED[4], K, W, bwt_layout=X2)),
            ("c5_quadfm", lambda: bench_fm(ctx, N5, 1, M5, L5, SEED[5], K, W, rank_queries=R5)),
            ("c5_quadfm_bwt16x2", lambda: bench_fm(ctx, N5, 1, M5, L5, SEED[5], K, W, bwt_layout=X2)),
            # the paper's FM workload shape: 150-bp reads at 1% substitutions from either
            # strand, each counted forward and reverse-complemented in one launch, over the configs[4] text
            ("c5_reads_150bp_both_strands", lambda: bench_fm(ctx, N5, 1, 10**7, 150, 55, K, W, strands=2, ptype=2)),
            # ... and at the paper's own genome size (3.1 Gbp block-repeat stand-in for CHM13v2; n+1 < 2^32)
            ("genome_scale_reads_3.1Gbp", lambda: bench_fm(ctx, 3_100_000_000, 1, 10**7, 150, 56, K, W, strands=2,
                                                           ptype=2)),
            ("c4_quadfm_approx1", lambda: bench_fm(ctx, N4, 0, 10**6, L4, SEED[4], K, W, kmax=1)),
            ("c4_quadfm_approx1_bwt16x2", lambda: bench_fm(ctx, N4, 0, 10**6, L4, SEED[4], K, W, kmax=1,
                                                           bwt_layout=X2)),
            ("c4_quadfm_approx2", lambda: bench_fm(ctx, N4, 0, 10**6, L4, SEED[4], K, W, kmax=2)),
            ("c4_quadfm_approx2_bwt16x2", lambda: bench_fm(ctx, N4, 0, 10**6, L4, SEED[4], K, W, kmax=2,
                                                           bwt_layout=X2)),
            # k = 3, the largest substitution count the API takes
            ("c4_quadfm_approx3", lambda: bench_fm(ctx, N4, 0, 2 * 10**5, L4, SEED[4], K, W, kmax=3)),
            ("c4_quadfm_approx3_bwt16x2", lambda: bench_fm(ctx, N4, 0, 2 * 10**5, L4, SEED[4], K, W, kmax=3,
                                                           bwt_layout=X2)),
            ("c5_reads_150bp_both_strands_approx1", lambda: bench_fm(ctx, N5, 1, 10**6, 150, 55, K, W, strands=2,
                                                                     kmax=1, ptype=2)),
            ("c5_reads_150bp_both_strands_approx2", lambda: bench_fm(ctx, N5, 1, 3 * 10**5, 150, 55, K, W, strands=2,
                                                                     kmax=2, ptype=2)),
            ("layout_variants", lambda: bench_variants(ctx, K, W)),
            ("latency_mode", lambda: bench_latency(ctx, K, W)),
            ("c1_small", lambda: bench_small(ctx, K, W)),
        ]
        only = set(args.only.split(",")) if args.only else None
        for name, fn in spec:
            if only is None or name in only:
                rows[name] = safe(ctx, fn)
    wall_gpu = time.perf_counter() - wall0
    ms = c2["ms"]
    value = c2["gq_s"]
    alg_bytes_q = BI_LINE_BYTES + 16
    achieved = alg_bytes_q * M2 / (ms * 1e-3) / 1e9          # per GPU, GB/s
    traffic, traffic_src = traffic_record(alg_bytes_q * M2)
    # the gather ceiling: the best measured launch shape loading exactly the lines rank loads
    ceil0 = max(c2[k]["gq_s"] for k in ("ceiling_mode0", "ceiling_mode3") if k in c2)
    if ctx.dist:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()
    clocks.stop()
    if ctx.rank != 0:
        return
    cpu = cpu_baselines(prep) if prep is not None else {}
    head_clk = clocks.window(*c2["_win"], full=True)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "Gqueries/s", "n_gpus": ctx.world, "steps": K,
        "warmup": W, "ms_per_step": round(ms, 4),
        "ms_per_step_median": round(c2["step_ms"]["median"], 4), "ms_per_step_min": round(c2["step_ms"]["min"], 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (seeded counter-based generators, gen/qrgen.h)",
        "config": workload_config(ctx.world),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": ("k_bi_rank2c (BiRank16 rank, Eq. 1; superblock words from 2-CTA cluster "
                                "shared memory)") if c2.get("smem_cache_cta_bytes") else "k_bi_rank2 (BiRank16 rank, Eq. 1)",
                     "alg_bytes_per_query": round(alg_bytes_q, 3), "peak_source": peak_src,
                     "gather_ceiling_gq_s": round(ceil0, 4), "frac_of_gather_ceiling": round(value / ceil0, 4)},
        "cpu_baseline": cpu.get("c2_rank"),
        "cpu_baseline_rows": {k: v for k, v in cpu.items() if k not in ("c2_rank", "host")},
        "cpu_host": cpu.get("host"),
        "e2e": finalize(c2.get("e2e"), clocks),
        "gpu_launches": c2["launches"],
        "clocks": head_clk,
        "checksum": c2["checksum"],
        "gather_ceiling": {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in c2.items() if k.startswith("ceiling")},
        "rows": finalize(rows, clocks),
        "wall_s": round(time.perf_counter() - wall0, 1), "wall_gpu_rows_s": round(wall_gpu, 1),
        "lib": qr.qr_version(),
    }
    print(json.dumps(line, default=lambda x: round(x, 4) if isinstance(x, float) else str(x)), flush=True)


if __name__ == "__main__":
    main()
