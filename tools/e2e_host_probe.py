"""e2e (host buffers) rank throughput on configs[1]: torch pinned buffers (cudaHostAlloc) vs
anonymous memory advised for transparent huge pages, touched, then cudaHostRegister'ed.  Run
after a host-memory-heavy job (e.g. the full-size tests) to see whether the page size of the
pinned buffers (IOMMU / DMA descriptor count) limits the PCIe rate."""
import ctypes, json, mmap, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2602_04103_b200 as qr  # noqa: E402

def thp():
    try:
        return open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
    except OSError:
        return "n/a"

def meminfo():
    d = {}
    for line in open("/proc/meminfo"):
        k, v = line.split(":", 1)
        if k in ("MemFree", "AnonHugePages", "HugePages_Total", "Hugepagesize"):
            d[k] = v.strip()
    return d

def thp_buffer(nbytes):
    mm = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    buf = (ctypes.c_char * len(mm)).from_buffer(mm)
    addr = ctypes.addressof(buf)
    off = (-addr) % (2 << 20)
    libc = ctypes.CDLL("libc.so.6", use_errno=True)
    libc.madvise(ctypes.c_void_p(addr + off), ctypes.c_size_t(nbytes), 14)   # MADV_HUGEPAGE
    a = np.frombuffer(mm, dtype=np.uint8, count=nbytes, offset=off).view(np.uint64)
    a[::512] = 0                                                              # touch every 4 KiB
    rt = torch.cuda.cudart()
    r = rt.cudaHostRegister(a.ctypes.data, nbytes, 0)
    return a, mm, buf, r

dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
print(json.dumps({"thp": thp(), "meminfo": meminfo()}), flush=True)
n, m = 1 << 34, 10**9
bits = torch.empty((n + 63) // 64, dtype=torch.uint64, device=dev)
gen.bits_dev(1, n, 0.5, bits)
h = qr.qr_birank_build(bits, n)
del bits
q = torch.empty(m, dtype=torch.uint64, device=dev)
gen.queries_dev(2, n, m, q)

def run(qh, oh):
    for _ in range(2):
        qr.qr_rank(h, qh, None, oh, m, st); st.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        qr.qr_rank(h, qh, None, oh, m, st); st.synchronize()
    return (time.perf_counter() - t0) / 3

for mode in ("torch_pinned", "thp_registered", "torch_pinned", "thp_registered"):
    if mode == "torch_pinned":
        qh = torch.empty(m, dtype=torch.uint64).pin_memory(); oh = torch.empty(m, dtype=torch.uint64).pin_memory()
        qh.copy_(q); keep = None
    else:
        qa, mq, bq, r1 = thp_buffer(8 * m); oa, mo, bo, r2 = thp_buffer(8 * m)
        qa[:] = q.cpu().numpy(); qh, oh = qa, oa; keep = (mq, bq, mo, bo)
    dt = run(qh, oh)
    print(json.dumps({"mode": mode, "ms": dt * 1e3, "gq_s": m / dt / 1e9, "meminfo": meminfo()}), flush=True)
    if mode == "thp_registered":
        rt = torch.cuda.cudart()
        rt.cudaHostUnregister(qa.ctypes.data); rt.cudaHostUnregister(oa.ctypes.data)
        del qa, oa, qh, oh
    else:
        del qh, oh
    torch.cuda.empty_cache()
