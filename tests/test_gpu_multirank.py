"""Multi-rank path on one GPU (gloo; the ranks' kernels never wait on each other): rank 0 builds,
broadcast_index replicates the layout, each rank answers its shard of the global query stream,
and the concatenated shards equal the oracle on the whole stream (shard invariance)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, layout, q):
    import torch
    import torch.distributed as dist

    import gen
    import paper_2602_04103_b200 as qr
    from paper_2602_04103_b200 import multigpu as mg

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        n, total = 3 * 63488 + 12345, 200003
        h0 = None
        if rank == 0:
            text = gen.bits(61, n) if layout in (qr.QR_LAYOUT_BIRANK16, qr.QR_LAYOUT_BIRANK64X2) else gen.dna(61, n)
            h0 = qr.qr_build(text, n, layout)
        h = mg.broadcast_index(h0, n, layout, dist, dev)
        i0, m = mg.shard(total, world, rank)
        qs, cs = gen.queries(62, n, m, i0=i0, with_c=True)
        out = torch.empty(m, dtype=torch.uint64, device=dev)
        sigma4 = layout in (qr.QR_LAYOUT_QUADRANK16, qr.QR_LAYOUT_QUADRANK64)
        qr.qr_rank(h, torch.from_numpy(qs).to(dev), torch.from_numpy(cs).to(dev) if sigma4 else None, out)
        torch.cuda.synchronize()
        q.put((rank, out.cpu().numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("layout", [1, 2, 3, 4])
def test_broadcast_replication_and_sharding(cuda, layout):
    import gen
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, layout, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, total = 3 * 63488 + 12345, 200003
    allq, allc = gen.queries(62, n, total, with_c=True)
    if layout in (1, 2):
        ref = oracle.BitsOracle(gen.bits(61, n), n).rank(allq)
    else:
        ref = oracle.DnaOracle(gen.dna(61, n), n).rank(allq, allc)
    got = np.concatenate([np.frombuffer(r[1], np.uint64) for r in res])
    assert np.array_equal(got, ref)


def test_gpu_local_cpus_and_affinity_restore(cuda):
    """The NUMA helper returns CPUs this process may use and always restores the affinity."""
    import os

    from paper_2602_04103_b200.multigpu import gpu_local_cpus, on_gpu_local_cpus

    before = os.sched_getaffinity(0)
    info = gpu_local_cpus(0)
    assert set(info["cpus"]) <= before and info["pci"].count(":") == 2
    with on_gpu_local_cpus(0) as inf:
        assert os.sched_getaffinity(0) <= before
        assert inf["pci"] == info["pci"]
    assert os.sched_getaffinity(0) == before
