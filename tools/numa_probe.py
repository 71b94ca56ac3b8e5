"""e2e (host buffers) rank throughput on configs[1] with the pinned buffers allocated from the
process's default CPUs vs from the CPUs local to the GPU (sysfs local_cpulist of its PCI
device), to see whether the host memory's NUMA node limits the PCIe transfer rate."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402
from paper_2602_04103_b200.multigpu import gpu_local_cpus  # noqa: E402

dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
bus = gpu_local_cpus(0)
print(json.dumps({"all_cpus": len(os.sched_getaffinity(0)), "gpu_local": bus}), flush=True)
n, m = 1 << 34, 10**9
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev)
gen.bits_dev(1, n, 0.5, bits)
h = qr.qr_birank_build(bits, n)
del bits
q = torch.empty(m, dtype=torch.uint64, device=dev)
gen.queries_dev(2, n, m, q)
allc = set(os.sched_getaffinity(0))
for mode in ("default", "local", "default", "local"):
    if mode == "local" and bus["cpus"]:
        os.sched_setaffinity(0, bus["cpus"])
    qh = torch.empty(m, dtype=torch.uint64).pin_memory()
    oh = torch.empty(m, dtype=torch.uint64).pin_memory()
    os.sched_setaffinity(0, allc)
    qh.copy_(q)
    for _ in range(2):
        qr.qr_rank(h, qh, None, oh, m, st); st.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        qr.qr_rank(h, qh, None, oh, m, st); st.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(json.dumps({"mode": mode, "ms": dt * 1e3, "gq_s": m / dt / 1e9}), flush=True)
    del qh, oh
    torch.cuda.empty_cache()
