"""PCIe ceiling for the staged host path: pinned H2D alone, D2H alone, and both directions at
once (two streams), 1 GiB each, CUDA events."""
import json, torch
dev = torch.device("cuda:0")
N = 1 << 30
h1 = torch.empty(N, dtype=torch.uint8).pin_memory(); h2 = torch.empty(N, dtype=torch.uint8).pin_memory()
d1 = torch.empty(N, dtype=torch.uint8, device=dev); d2 = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
r = {"h2d_gbs": N / timed(h2d) / 1e6, "d2h_gbs": N / timed(d2h) / 1e6}
ms = timed(both)
r["bidir_each_gbs"] = N / ms / 1e6
print(json.dumps(r))
