"""Cost of mapping / unmapping large device allocations: cudaMalloc vs the stream-ordered pool."""
import json, time
import cuda.bindings.runtime as rt

def ck(r):
    if isinstance(r, tuple):
        assert r[0] == rt.cudaError_t.cudaSuccess, r
        return r[1] if len(r) > 1 else None
    assert r == rt.cudaError_t.cudaSuccess, r

ck(rt.cudaSetDevice(0)); ck(rt.cudaFree(0))
st = ck(rt.cudaStreamCreate())
for total_gb in (4, 16, 43):
    for parts in (1, 10):
        sz = total_gb * (1 << 30) // parts
        for kind in ("malloc", "async"):
            t0 = time.perf_counter()
            ptrs = []
            for _ in range(parts):
                ptrs.append(ck(rt.cudaMalloc(sz)) if kind == "malloc" else ck(rt.cudaMallocAsync(sz, st)))
            ck(rt.cudaStreamSynchronize(st)); t1 = time.perf_counter()
            for p in ptrs:
                ck(rt.cudaFree(p)) if kind == "malloc" else ck(rt.cudaFreeAsync(p, st))
            ck(rt.cudaStreamSynchronize(st)); t2 = time.perf_counter()
            print(json.dumps({"gb": total_gb, "parts": parts, "kind": kind, "alloc_s": round(t1 - t0, 4),
                              "free_s": round(t2 - t1, 4)}), flush=True)
