"""The multi-GPU path over NCCL across two real devices; skipped below 2 GPUs
(the gpurun boxes and the driver's round-end tests have one).  Rank 0 builds, broadcast_index
replicates the layout over NCCL (NVLink / NVSwitch on a B200 box), qr_clone_to_device copies it
peer to peer, every rank answers its shard of the global query / pattern streams, the shards
concatenate to the oracle's answers, and the per-rank output checksums (qr_checksum) summed with
one u64 all_reduce equal the one-GPU checksum of the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import gen
    import paper_2602_04103_b200 as qr
    from paper_2602_04103_b200 import multigpu as mg

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        n, total = 5 * 63488 + 321, 400009
        h0 = qr.qr_birank_build(gen.bits(81, n), n, device=0) if rank == 0 else None
        h = mg.broadcast_index(h0, n, qr.QR_LAYOUT_BIRANK16, dist, dev)
        i0, m = mg.shard(total, world, rank)
        qd = torch.empty(m, dtype=torch.uint64, device=dev)
        gen.queries_dev(82, n, m, qd, i0=i0)
        out = torch.empty_like(qd)
        qr.qr_rank(h, qd, None, out)
        acc = torch.zeros(1, dtype=torch.uint64, device=dev)
        qr.qr_checksum(out, m, 8, i0, acc)
        torch.cuda.synchronize()
        c_all = mg.reduce_sum_u64(int(acc.view(torch.int64).item()), dist, dev)
        # peer-to-peer clone of rank 0's replica onto this rank's device answers identically
        hc = qr.qr_clone_to_device(h, rank)
        out2 = torch.empty_like(qd)
        qr.qr_rank(hc, qd, None, out2)
        torch.cuda.synchronize()
        # QuadFm: every rank builds the index from the seeded text and counts its shard
        nf = 200000
        t = torch.empty((nf + 31) // 32 + 1, dtype=torch.uint64, device=dev)
        gen.dna_dev(83, nf, 0, t)
        fm = qr.qr_fm_build(t, nf, device=rank)
        j0, mf = mg.shard(20000, world, rank)
        pats = torch.empty(mf * 32, dtype=torch.uint8, device=dev)
        gen.patterns_dev(84, 0, mf, 32, t, nf, pats, i0=j0)
        cnt = torch.empty(mf, dtype=torch.int32, device=dev)
        qr.qr_fm_count(fm, pats, None, 32, cnt, mf)
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy().tobytes(), bool(torch.equal(out, out2)), c_all,
               cnt.cpu().numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_nccl_two_gpus_replicate_shard_checksum(cuda):
    if torch.cuda.device_count() < WORLD:
        pytest.skip(f"needs {WORLD} GPUs, this box has {torch.cuda.device_count()}")
    import gen
    import oracle
    import paper_2602_04103_b200 as qr

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n, total = 5 * 63488 + 321, 400009
    allq = gen.queries(82, n, total)
    ref = oracle.BitsOracle(gen.bits(81, n), n).rank(allq)
    assert np.array_equal(np.concatenate([np.frombuffer(r[1], np.uint64) for r in res]), ref)
    assert all(r[2] for r in res)
    # the one-GPU checksum of the whole batch equals the all_reduce of the shards'
    acc = torch.zeros(1, dtype=torch.uint64, device=cuda)
    qr.qr_checksum(torch.from_numpy(ref).to(cuda), total, 8, 0, acc)
    torch.cuda.synchronize()
    whole = int(acc.view(torch.int64).item()) & ((1 << 64) - 1)
    assert all(r[3] == whole for r in res)
    nf = 200000
    sym = gen.unpack_dna(gen.dna(83, nf, 0), nf)
    pats = gen.patterns(84, 0, 20000, 32, gen.dna(83, nf, 0), nf)
    fref = oracle.FmOracle(sym).count(pats, np.arange(20000, dtype=np.uint64) * 32, np.full(20000, 32, np.uint32))
    assert np.array_equal(np.concatenate([np.frombuffer(r[4], np.uint32) for r in res]), fref)
