"""Multi-rank host logic on CPU (gloo, world size 2): shards partition the global index
space, per-rank generated shards concatenate to the global stream (shard invariance of the
inputs), and the max/sum reductions and the weak-scaling throughput arithmetic are right."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_2602_04103_b200 import multigpu as mg


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, total = 10**6, 100003
        i0, m = mg.shard(total, world, rank)
        qs = gen.queries(5, n, m, i0=i0)
        w = gen.bits(5, n)
        out = oracle.BitsOracle(w, n).rank(qs)                   # stand-in for the per-GPU kernel
        t_ms = 10.0 + rank                                       # per-rank "kernel time"
        mx = mg.reduce_max(t_ms, dist)
        tot = mg.reduce_sum(m, dist)
        chk = mg.reduce_sum(int(np.bitwise_xor.reduce(out) & 0x7FFFFFFF), dist)
        # u64 checksums near 2^64 wrap exactly; every rank sees every rank's value in order
        big = (1 << 64) - 1 - rank
        c64 = mg.reduce_sum_u64(big, dist)
        allv = mg.gather_u64(big * 3 + rank, dist)
        q.put((rank, i0, m, qs.tobytes(), out.tobytes(), mx, tot, chk, c64, allv))
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for total in (0, 1, 7, 10**9 + 3):
        for world in (1, 2, 3, 8):
            pieces = [mg.shard(total, world, r) for r in range(world)]
            assert pieces[0][0] == 0
            assert sum(c for _, c in pieces) == total
            for (a, ca), (b, _) in zip(pieces, pieces[1:]):
                assert a + ca == b
    assert mg.weak_shard(10**9, 3) == (3 * 10**9, 10**9)
    assert mg.throughput(8 * 10**9, 250.0) == 32e9


def test_two_rank_gloo_shard_invariance():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, total = 10**6, 100003
    allq = gen.queries(5, n, total)
    cat_q = np.concatenate([np.frombuffer(r[3], np.uint64) for r in res])
    assert np.array_equal(cat_q, allq)                          # shards = the global stream
    ref = oracle.BitsOracle(gen.bits(5, n), n).rank(allq)
    cat_o = np.concatenate([np.frombuffer(r[4], np.uint64) for r in res])
    assert np.array_equal(cat_o, ref)                           # per-rank outputs concatenate
    assert all(r[5] == 11.0 for r in res)                       # max over ranks
    assert all(r[6] == total for r in res)
    assert res[0][7] == res[1][7]
    M = (1 << 64) - 1
    assert all(r[8] == (2 * M - 1) % (1 << 64) for r in res)
    assert all(r[9] == [((M - k) * 3 + k) % (1 << 64) for k in range(2)] for r in res)
    assert mg.reduce_sum_u64(M + 5) == 4 and mg.gather_u64(7) == [7]      # one rank: identity (mod 2^64)


def test_parse_cpulist():
    from paper_2602_04103_b200.multigpu import parse_cpulist

    assert parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert parse_cpulist("5") == {5}
    assert parse_cpulist("") == set()
