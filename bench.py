#!/usr/bin/env python
"""Benchmark of the hot path on B200 (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--rows all|headline]

Headline (`value`): BiRank16 rank queries/s on configs[1] (n = 2^34 bits, p = 0.5, 10^9 queries
per GPU, u64 out), whole job over N GPUs (weak scaling: each GPU keeps its 10^9 queries),
CUDA-event time on the launching stream, max over ranks.  `rows` adds every other §8(a) row
measured in the same run (gather ceiling, p = 0.01, QuadRank rank / rank_all4 on configs[2],
QuadFm count on configs[3] and configs[4], the small configs[0]).  Inputs are created on the
device from the seeded generators before the timed region; every timed input (the line array
2.2 GB, the query array 8 GB) is far larger than the 126 MB L2, so no flush is needed.

--impl reference: the CPU oracle (oracle/, plain C, OpenMP over queries) timed on the host
cores on a bounded sample of the same workload each step; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rank Gqueries/s & HBM gather GB/s vs roofline; QuadFm patterns/s @1/2/4/8"
N2, M2 = 1 << 34, 10**9                 # configs[1]
N3, M3 = 1 << 32, 10**9                 # configs[2]
N4, M4, L4 = 1 << 26, 10**7, 32         # configs[3]
N5, M5, L5 = 1 << 30, 10**8, 100        # configs[4] (patterns; rank queries: 10^9 per GPU shard)
N1, M1 = 1 << 20, 10**6                 # configs[0]
SEED = {1: 1, 2: 2, 3: 3, 4: 4, 5: 5}
# expected bytes of one BiRank query: sector 0 always, sector 1 when the
# query lies right of the anchor (data bits [240,496): 256/496 of uniform q) + 8 B q + 8 B out
BI_LINE_BYTES = 32 + 32 * 256 / 496
QD_LINE_BYTES = 32 + 32 * 128 / 224     # data chars [96,224) of 224 need sector 1


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,temperature.gpu,temperature.memory,clocks.mem,serial")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

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
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons, tg, tm, mem, serial = [], None, set(), [], [], [], None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for k, name in enumerate(names):
                if p[5 + k].lower().startswith("active"):
                    reasons.add(name)
            for lst, k in ((tg, 9), (tm, 10), (mem, 11)):       # GPU / HBM temperature, memory clock
                try:
                    lst.append(float(p[k]))
                except (ValueError, IndexError):
                    pass
            if len(p) > 12:
                serial = p[12]
        os.unlink(self.path)
        med = lambda v: statistics.median(v) if v else None   # noqa: E731
        return {"sm_mhz": med(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "gpu_temp_c": med(tg), "hbm_temp_c": med(tm), "mem_mhz": med(mem), "gpu_serial": serial}


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

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, x: int) -> int:
        if not self.dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.int64, device=self.dev)
        self.dist.all_reduce(t)
        return int(t.item())

    def timed(self, fn, steps: int, warmup: int, clocks: Clocks | None = None) -> float:
        """ms per step: W warm-up calls, then EXACTLY K calls bracketed by barrier + synchronize,
        CUDA events on the launching stream, max over ranks."""
        torch = self.torch
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        self.barrier()
        torch.cuda.synchronize()
        if clocks:
            clocks.start()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record(self.stream)
        for i in range(steps):
            fn()
            ev[i + 1].record(self.stream)
        torch.cuda.synchronize()
        self.barrier()
        ms = ev[0].elapsed_time(ev[-1]) / steps
        # per-step times (median and minimum beside the mean), kept for the caller
        per = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(steps))
        self.last_step_ms = {"median": self.max_over_ranks(per[len(per) // 2]), "min": self.max_over_ranks(per[0])}
        return self.max_over_ranks(ms)


def shard(total, world, rank):
    """contiguous shard of a global index range (paper_2602_04103_b200.multigpu.shard), imported
    lazily: the product package loads libqrank.so on import, which the reference arm must not."""
    from paper_2602_04103_b200.multigpu import shard as _shard

    return _shard(total, world, rank)


# ------------------------------------------------------------------ rows
def bench_birank(ctx, p: float, steps, warmup, with_ceiling: bool, clocks=None, e2e=False):
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    if ctx.dist and ctx.args.replicate == "broadcast":
        # rank 0 builds; the layout is broadcast to every rank (NCCL over NVLink) and imported
        from paper_2602_04103_b200.multigpu import broadcast_index

        h0 = None
        if ctx.rank == 0:
            bits = torch.empty((N2 + 63) // 64, dtype=torch.uint64, device=ctx.dev)
            gen.bits_dev(SEED[2] if p == 0.5 else 22, N2, p, bits)
            h0 = qr.qr_birank_build(bits, N2, device=ctx.gpu)
            del bits
        h = broadcast_index(h0, N2, qr.QR_LAYOUT_BIRANK16, ctx.dist, ctx.dev)
    else:
        bits = torch.empty((N2 + 63) // 64, dtype=torch.uint64, device=ctx.dev)
        gen.bits_dev(SEED[2] if p == 0.5 else 22, N2, p, bits)
        h = qr.qr_birank_build(bits, N2, device=ctx.gpu)
        del bits
    m = M2                                         # per GPU (weak scaling)
    i0 = ctx.rank * m
    q = torch.empty(m, dtype=torch.uint64, device=ctx.dev)
    gen.queries_dev(SEED[2], N2, m, q, i0=i0)
    out = torch.empty_like(q)
    torch.cuda.synchronize()
    ms = ctx.timed(lambda: qr.qr_rank(h, q, None, out, m, ctx.stream), steps, warmup, clocks)
    clk = clocks.stop() if clocks else None
    res = {"ms": ms, "m_per_gpu": m, "gq_s": ctx.world * m / ms / 1e6, "launches": steps, "clocks": clk,
           "step_ms": dict(ctx.last_step_ms)}
    res["smem_cache_cta_bytes"] = qr.qr_super_cache_bytes(h)
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
                      "ms_per_step_max": round(max(step_wall), 3)}
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
    return {"ms": ms, "gq_s": ctx.world * m / ms / 1e6, "n_bits": n}


def bench_quadrank(ctx, steps, warmup):
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    text = torch.empty((N3 + 31) // 32, dtype=torch.uint64, device=ctx.dev)
    gen.dna_dev(SEED[3], N3, 0, text)
    h = qr.qr_quadrank_build(text, N3, device=ctx.gpu)
    del text
    m = M3
    q = torch.empty(m, dtype=torch.uint64, device=ctx.dev)
    c = torch.empty(m, dtype=torch.uint8, device=ctx.dev)
    gen.queries_dev(SEED[3], N3, m, q, c, i0=ctx.rank * m)
    out = torch.empty_like(q)
    ms = ctx.timed(lambda: qr.qr_rank(h, q, c, out, m, ctx.stream), steps, warmup)
    cms = ctx.timed(lambda: qr.qr_gather_ceiling(h, q, out, 0, m, ctx.stream), steps, warmup)
    del out
    out4 = torch.empty((m, 4), dtype=torch.uint64, device=ctx.dev)
    ms4 = ctx.timed(lambda: qr.qr_rank_all4(h, q, out4, m, ctx.stream), steps, warmup)
    # rank_4's own ceiling: the same loads with its 32-B output stream (qr_gather_ceiling mode 4)
    cms4 = ctx.timed(lambda: qr.qr_gather_ceiling(h, q, out4, 4, m, ctx.stream), steps, warmup)
    del q, c, out4
    h.free()
    torch.cuda.empty_cache()
    return {"rank": {"ms": ms, "gq_s": ctx.world * m / ms / 1e6},
            "ceiling_mode0": {"ms": cms, "gq_s": ctx.world * m / cms / 1e6},
            "rank_all4": {"ms": ms4, "gq_s": ctx.world * m / ms4 / 1e6},
            "ceiling_rank4_shape": {"ms": cms4, "gq_s": ctx.world * m / cms4 / 1e6}}


def bench_fm(ctx, n, kind, m_total, length, seed, steps, warmup, rank_queries=0, bwt_layout=None):
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=ctx.dev)
    gen.dna_dev(seed, n, kind, text)
    t0 = time.perf_counter()
    fm = qr.qr_fm_build(text, n, device=ctx.gpu, bwt_layout=bwt_layout)
    build_s = time.perf_counter() - t0
    i0, m = shard(m_total, ctx.world, ctx.rank)
    pats = torch.empty(m * length, dtype=torch.uint8, device=ctx.dev)
    gen.patterns_dev(seed, 0 if kind == 0 else 1, m, length, text, n, pats, i0=i0)
    out = torch.empty(m, dtype=torch.int32, device=ctx.dev)
    work = torch.zeros(2, dtype=torch.uint64, device=ctx.dev)
    qr.qr_fm_count_work(fm, pats, None, length, out, m, work, ctx.stream)
    torch.cuda.synchronize()
    steps_done, lines = (int(x) for x in work.cpu())
    ms = ctx.timed(lambda: qr.qr_fm_count(fm, pats, None, length, out, m, ctx.stream), steps, warmup)
    lines_all = ctx.sum_over_ranks(lines)
    res = {"ms": ms, "patterns_per_s": m_total / ms * 1e3, "build_s": round(build_s, 3),
           "steps_per_pattern": steps_done / max(m, 1), "lines_per_pattern": lines / max(m, 1),
           "lines_per_s": lines_all / ms * 1e3,
           "alg_gbs": (lines_all * 64 + m_total * (length + 4)) / ms / 1e6}
    del pats, out
    if rank_queries:
        q = torch.empty(rank_queries, dtype=torch.uint64, device=ctx.dev)
        c = torch.empty(rank_queries, dtype=torch.uint8, device=ctx.dev)
        gen.queries_dev(seed, n + 1, rank_queries, q, c, i0=ctx.rank * rank_queries)
        o = torch.empty_like(q)
        rms = ctx.timed(lambda: qr.qr_rank(fm.bwt, q, c, o, rank_queries, ctx.stream), steps, warmup)
        res["rank"] = {"ms": rms, "gq_s": ctx.world * rank_queries / rms / 1e6, "m_per_gpu": rank_queries}
        del q, c, o
    fm.free()
    del text
    torch.cuda.empty_cache()
    return res


def bench_reads_safe(ctx, n, m_total, length, seed, steps, warmup):
    try:
        ctx.torch.cuda.empty_cache()
        return bench_reads(ctx, n, m_total, length, seed, steps, warmup)
    except Exception as e:                          # e.g. out of memory on a smaller GPU
        ctx.torch.cuda.empty_cache()
        return {"skipped": str(e)[:200]}


def bench_reads(ctx, n, m_total, length, seed, steps, warmup):
    """The paper's FM workload shape: 150-bp reads with 1% substitutions from
    either strand, each counted in both directions in one launch (qr_fm_count_both), over the
    configs[4] block-repeat text (stand-in for CHM13v2)."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=ctx.dev)
    gen.dna_dev(seed, n, 1, text)
    t0 = time.perf_counter()
    fm = qr.qr_fm_build(text, n, device=ctx.gpu)
    build_s = time.perf_counter() - t0
    i0, m = shard(m_total, ctx.world, ctx.rank)
    pats = torch.empty(m * length, dtype=torch.uint8, device=ctx.dev)
    gen.patterns_dev(seed, 2, m, length, text, n, pats, i0=i0)
    of = torch.empty(m, dtype=torch.int32, device=ctx.dev)
    orc = torch.empty(m, dtype=torch.int32, device=ctx.dev)
    ms = ctx.timed(lambda: qr.qr_fm_count_both(fm, pats, None, length, of, orc, m, ctx.stream), steps, warmup)
    hit = int(((of > 0) | (orc > 0)).sum())
    fm.free()
    del text, pats, of, orc
    torch.cuda.empty_cache()
    return {"ms": ms, "reads_per_s": m_total / ms * 1e3, "searches_per_s": 2 * m_total / ms * 1e3,
            "read_len": length, "reads": m_total, "frac_reads_matching": hit / max(m, 1), "text_len": n,
            "fm_build_s": round(build_s, 2)}


def bench_reads_approx(ctx, n, m_total, length, seed, steps, warmup, kmax):
    """The paper's read workload (150 bp, 1% substitutions, either strand) counted
    within kmax substitutions on both strands in one launch (qr_fm_count_approx_both)."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=ctx.dev)
    gen.dna_dev(5, n, 1, text)
    fm = qr.qr_fm_build(text, n, device=ctx.gpu)
    i0, m = shard(m_total, ctx.world, ctx.rank)
    pats = torch.empty(m * length, dtype=torch.uint8, device=ctx.dev)
    gen.patterns_dev(seed, 2, m, length, text, n, pats, i0=i0)
    of = torch.empty(m, dtype=torch.int32, device=ctx.dev)
    orc = torch.empty_like(of)
    ms = ctx.timed(lambda: qr.qr_fm_count_approx_both(fm, pats, None, length, kmax, of, orc, m, ctx.stream), steps,
                   warmup)
    hit = int(((of > 0) | (orc > 0)).sum())
    fm.free()
    del text, pats, of, orc
    torch.cuda.empty_cache()
    return {"ms": ms, "reads_per_s": m_total / ms * 1e3, "searches_per_s": 2 * m_total / ms * 1e3,
            "max_mismatches": kmax, "read_len": length, "reads": m_total, "frac_reads_matching": hit / max(m, 1),
            "text_len": n}


def bench_approx(ctx, n, m_total, length, seed, steps, warmup, bwt_layout=None, kmax=1):
    """<=kmax-substitution counting (rank_4-driven, NEXT §8(f)3) on the configs[3] text/patterns."""
    import gen
    import paper_2602_04103_b200 as qr

    torch = ctx.torch
    text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=ctx.dev)
    gen.dna_dev(seed, n, 0, text)
    fm = qr.qr_fm_build(text, n, device=ctx.gpu, bwt_layout=bwt_layout)
    i0, m = shard(m_total, ctx.world, ctx.rank)
    pats = torch.empty(m * length, dtype=torch.uint8, device=ctx.dev)
    gen.patterns_dev(seed, 0, m, length, text, n, pats, i0=i0)
    out = torch.empty(m, dtype=torch.int32, device=ctx.dev)
    ms = ctx.timed(lambda: qr.qr_fm_count_approx(fm, pats, None, length, kmax, out, m, ctx.stream), steps, warmup)
    fm.free()
    del text, pats, out
    torch.cuda.empty_cache()
    return {"ms": ms, "patterns_per_s": m_total / ms * 1e3, "max_mismatches": kmax, "patterns": m_total,
            "pattern_len": length}


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
                    "overhead": (h.line_bytes + h.super_bytes) / (N2 / 8) - 1}
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
        ms4 = ctx.timed(lambda: qr.qr_rank_all4(h, q, o4, M3, ctx.stream), steps, warmup)
        res[key] = {"rank": {"ms": ms, "gq_s": ctx.world * M3 / ms / 1e6},
                    "rank_all4": {"ms": ms4, "gq_s": ctx.world * M3 / ms4 / 1e6},
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
        L2, chains2 = 200, 148 * 2048                  # many chains: latency-bound throughput
        m2 = L2 * chains2
        q2 = torch.empty(m2, dtype=torch.uint64, device=ctx.dev)
        gen.queries_dev(SEED[2] + 1, N2, m2, q2)
        out2 = torch.empty_like(q2)
        ms2 = ctx.timed(lambda: qr.qr_rank_chain(h, q2, None, out2, L2, m2, ctx.stream), max(2, steps // 2), warmup)
        res[name] = {"ns_per_dependent_query": ms * 1e6 / L, "chains": chains, "chain_len": L,
                     "many_chains_gq_s": m2 / ms2 / 1e6, "many_chains": chains2}
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
    return {"ms": ms, "gq_s": ctx.world * M1 / ms / 1e6}


# ------------------------------------------------------------------ CPU oracle
def cpu_oracle_rank(target_s: float = 10.0, per_step_q: int | None = None):
    """The oracle (as it stands) on the host cores: BiRank config 2 text regenerated on the
    host, plain prefix array, rank on a bounded sample of the same query stream."""
    import numpy as np

    import gen
    import oracle

    t0 = time.perf_counter()
    words = gen.bits(SEED[2], N2, 0.5)
    ora = oracle.BitsOracle(words, N2)
    prep = time.perf_counter() - t0
    m = 1 << 21
    q = gen.queries(SEED[2], N2, m)
    t0 = time.perf_counter()
    ora.rank(q)
    dt = time.perf_counter() - t0
    if per_step_q is None:
        per_step_q = int(min(2e8, max(m, m * target_s / max(dt, 1e-6))))
    q = gen.queries(SEED[2], N2, per_step_q)
    return ora, q, prep


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
            "repo_so_loaded": repo_so_loaded()}
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", default="all", choices=["all", "headline"])
    ap.add_argument("--no-cpu", action="store_true")
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
    K, W = args.steps, max(3, args.warmup)
    peak, peak_src = peaks()
    clocks = Clocks(ctx.gpu)
    wall0 = time.perf_counter()
    c2 = bench_birank(ctx, 0.5, K, W, with_ceiling=True, clocks=clocks, e2e=True)
    rows = {}
    if args.rows == "all":
        rows["c2_p0.01"] = bench_birank(ctx, 0.01, K, W, with_ceiling=False)
        rows["birank16_2^35_paper_size"] = bench_birank_size(ctx, 35, K, W)
        rows["c3_quadrank"] = bench_quadrank(ctx, K, W)
        rows["c4_quadfm"] = bench_fm(ctx, N4, 0, M4, L4, SEED[4], K, W)
        rows["c5_quadfm"] = bench_fm(ctx, N5, 1, M5, L5, SEED[5], K, W, rank_queries=10**9)
        # the same searches over the sector-local QuadRank16x2 BWT (B200 variant)
        rows["c4_quadfm_bwt16x2"] = bench_fm(ctx, N4, 0, M4, L4, SEED[4], K, W, bwt_layout=qr.QR_LAYOUT_QUADRANK16X2)
        rows["c5_quadfm_bwt16x2"] = bench_fm(ctx, N5, 1, M5, L5, SEED[5], K, W, bwt_layout=qr.QR_LAYOUT_QUADRANK16X2)
        rows["c5_reads_150bp_both_strands"] = bench_reads(ctx, N5, 10**7, 150, 55, K, W)
        # the paper's FM workload at its own scale: a 3.1 Gbp text (block-repeat
        # stand-in for CHM13v2; n+1 < 2^32), 150-bp reads at 1% substitutions, both strands
        rows["genome_scale_reads_3.1Gbp"] = bench_reads_safe(ctx, 3_100_000_000, 10**7, 150, 56, K, W)
        rows["c4_quadfm_approx1"] = bench_approx(ctx, N4, 10**6, L4, SEED[4], K, W)
        rows["c4_quadfm_approx1_bwt16x2"] = bench_approx(ctx, N4, 10**6, L4, SEED[4], K, W,
                                                         bwt_layout=qr.QR_LAYOUT_QUADRANK16X2)
        rows["c4_quadfm_approx2"] = bench_approx(ctx, N4, 10**6, L4, SEED[4], K, W, kmax=2)
        rows["c5_reads_150bp_both_strands_approx1"] = bench_reads_approx(ctx, N5, 10**6, 150, 55, K, W, 1)
        rows["c5_reads_150bp_both_strands_approx2"] = bench_reads_approx(ctx, N5, 3 * 10**5, 150, 55, K, W, 2)
        rows["layout_variants"] = bench_variants(ctx, K, W)
        rows["latency_mode"] = bench_latency(ctx, K, W)
        rows["c1_small"] = bench_small(ctx, K, W)
    ms = c2["ms"]
    value = c2["gq_s"]
    alg_bytes_q = BI_LINE_BYTES + 16
    achieved = alg_bytes_q * M2 / (ms * 1e-3) / 1e9          # per GPU, GB/s
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get("k_bi_rank_bytes_per_launch")
    except Exception:
        pass
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        import oracle

        oracle.set_threads(len(os.sched_getaffinity(0)))
        ora, q, prep = cpu_oracle_rank(per_step_q=1 << 27)
        t0 = time.perf_counter()
        reps = 0
        while True:                                # ~10 s of CPU work on the bounded sample
            ora.rank(q)
            reps += 1
            if time.perf_counter() - t0 > 10.0:
                break
        dt = time.perf_counter() - t0
        cpu = {"value": round(reps * q.size / dt / 1e9, 6), "unit": "Gqueries/s", "cores": oracle.threads(),
               "kind": "oracle",
               "sample": f"{q.size} queries of the configs[1] stream x {reps} passes ({dt:.1f}s of CPU work); "
                         f"host-regenerated text 2^34 bits, plain prefix-array precompute {prep:.1f}s untimed"}
    # the gather ceiling: the best measured launch shape loading exactly the lines rank loads
    ceil0 = max(c2[k]["gq_s"] for k in ("ceiling_mode0", "ceiling_mode3") if k in c2)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "Gqueries/s", "n_gpus": ctx.world, "steps": K,
        "warmup": W, "ms_per_step": round(ms, 4),
        "ms_per_step_median": round(c2["step_ms"]["median"], 4), "ms_per_step_min": round(c2["step_ms"]["min"], 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic (seeded counter-based generators, gen/qrgen.h)",
        "config": workload_config(ctx.world),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": ("k_bi_rank2c (BiRank16 rank, Eq. 1; superblock words from 2-CTA cluster "
                                "shared memory)") if c2.get("smem_cache_cta_bytes") else "k_bi_rank2 (BiRank16 rank, Eq. 1)",
                     "alg_bytes_per_query": round(alg_bytes_q, 3), "peak_source": peak_src,
                     "gather_ceiling_gq_s": round(ceil0, 4), "frac_of_gather_ceiling": round(value / ceil0, 4)},
        "cpu_baseline": cpu,
        "e2e": c2.get("e2e"),
        "gpu_launches": c2["launches"],
        "clocks": c2["clocks"],
        "gather_ceiling": {k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in c2.items() if k.startswith("ceiling")},
        "rows": rows,
        "wall_s": round(time.perf_counter() - wall0, 1),
        "lib": qr.qr_version(),
    }
    if ctx.rank == 0:
        print(json.dumps(line, default=lambda x: round(x, 4) if isinstance(x, float) else str(x)), flush=True)
    if ctx.dist:
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
