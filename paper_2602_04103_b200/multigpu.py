"""Single-box multi-GPU driver pieces: replicate the structure, shard the
queries/patterns, no data-path collective.

Every query and pattern is independent, so rank r of W takes the
contiguous global index range [r*M/W, (r+1)*M/W) and generates it locally from
(seed, global index); the only collectives are the max of the per-rank kernel times and
the sum of per-rank counters at the end (torch.distributed: NCCL on GPUs, gloo in tests).
"""
from __future__ import annotations


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first global index, count) of rank's contiguous share of `total` items."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi - lo


def weak_shard(per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank keeps `per_rank` items; rank r owns [r*per_rank, (r+1)*per_rank)."""
    return rank * per_rank, per_rank


def reduce_max(x: float, dist=None, device=None) -> float:
    """max over ranks of a per-rank time (the job time of a data-parallel step)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: int, dist=None, device=None) -> int:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return int(x)
    import torch

    t = torch.tensor([int(x)], dtype=torch.int64, device=device)
    dist.all_reduce(t)
    return int(t.item())


def reduce_sum_u64(x: int, dist=None, device=None) -> int:
    """sum mod 2^64 of one u64 per rank (an output checksum): all_reduce of the
    two 32-bit halves in int64, which cannot overflow for up to 2^31 ranks, then recombined."""
    x &= (1 << 64) - 1
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    import torch

    t = torch.tensor([x & 0xFFFFFFFF, x >> 32], dtype=torch.int64, device=device)
    dist.all_reduce(t)
    lo, hi = (int(v) for v in t.cpu())
    return (lo + (hi << 32)) & ((1 << 64) - 1)


def gather_u64(x: int, dist=None, device=None) -> list:
    """every rank's u64 (e.g. its shard checksum), in rank order, on every rank."""
    x &= (1 << 64) - 1
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [x]
    import torch

    t = torch.tensor([x & 0xFFFFFFFF, x >> 32], dtype=torch.int64, device=device)
    outs = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(outs, t)
    return [int(o[0]) + (int(o[1]) << 32) for o in outs]


def throughput(units_all_ranks: int, max_ms: float) -> float:
    """whole-job units per second: all ranks' units over the slowest rank's time."""
    return units_all_ranks / (max_ms * 1e-3)


def replicate(handle, device: int, stream=None):
    """Copy a built BiRank/QuadRank handle to another GPU (peer copy over NVLink/NVSwitch)."""
    from . import qr_clone_to_device

    return qr_clone_to_device(handle, device, stream)


def broadcast_index(h, n: int, layout: int, dist, device, src: int = 0):
    """Replicate a rank structure over the process group: rank `src` exports its layout into
    device buffers, one broadcast per buffer over NCCL (NVLink / NVSwitch on a B200 box), every
    other rank imports it (`h` is ignored there and may be None).  Returns the local handle."""
    import torch

    from . import _check, _ptr, lib, qr_import_layout

    rank = dist.get_rank()
    device = torch.device("cuda", device_index(device))
    if rank == src:
        sizes = torch.tensor([h.line_bytes, h.super_bytes], dtype=torch.int64, device=device)
    else:
        sizes = torch.zeros(2, dtype=torch.int64, device=device)
    dist.broadcast(sizes, src)
    lb, sb = (int(x) for x in sizes.cpu())
    lines = torch.empty(lb, dtype=torch.uint8, device=device)
    sup = torch.empty(max(sb, 1), dtype=torch.uint8, device=device)
    if rank == src:
        _check(lib().qr_export_layout(h.ptr, _ptr(lines), _ptr(sup) if sb else None), "qr_export_layout")
    dist.broadcast(lines, src)
    if sb:
        dist.broadcast(sup, src)
    torch.cuda.synchronize(device)
    if rank == src:
        return h
    return qr_import_layout(lines, sup[:sb] if sb else None, n, layout, device=device_index(device))


def device_index(device) -> int:
    """CUDA ordinal of an int, a "cuda:k" string or a torch.device; "cuda" without an index is the
    current device."""
    import torch

    if isinstance(device, int):
        return device
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"not a CUDA device: {device}")
    return d.index if d.index is not None else torch.cuda.current_device()


def parse_cpulist(text: str) -> set:
    """CPU ids of a Linux cpulist string ("0-7,16-23,40")."""
    cpus = set()
    for part in text.strip().split(","):
        part = part.strip()
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


def gpu_local_cpus(device: int = 0) -> dict:
    """CPUs and NUMA node local to a GPU's PCI device (sysfs), intersected with the CPUs this
    process may run on.  Pinned host buffers allocated while running there land on the GPU's
    node, so host<->device copies do not cross the socket interconnect."""
    import torch

    p = torch.cuda.get_device_properties(device)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    base = f"/sys/bus/pci/devices/{bus}"
    cpus, node = set(), -1
    try:
        with open(f"{base}/local_cpulist") as f:
            cpus = parse_cpulist(f.read())
        with open(f"{base}/numa_node") as f:
            node = int(f.read().strip())
    except (OSError, ValueError):
        pass
    import os

    cpus &= set(os.sched_getaffinity(0))
    return {"pci": bus, "numa_node": node, "cpus": sorted(cpus)}


class on_gpu_local_cpus:
    """Context manager: run the block on the GPU-local CPUs (e.g. while allocating pinned host
    memory), then restore the previous affinity.  A no-op when sysfs has no locality data."""

    def __init__(self, device: int = 0):
        self.device = device

    def __enter__(self):
        import os

        self.prev = os.sched_getaffinity(0)
        self.info = gpu_local_cpus(self.device)
        if self.info["cpus"] and len(self.info["cpus"]) < len(self.prev):
            os.sched_setaffinity(0, self.info["cpus"])
        return self.info

    def __exit__(self, *exc):
        import os

        os.sched_setaffinity(0, self.prev)
        return False
