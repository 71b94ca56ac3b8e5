cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fm.py -q --timeout 1200 -x -rf -k "approx or work_order" > gpurun_out/pytest_fm.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fm.log
cat > /tmp/approx_probe.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, gen, paper_2602_04103_b200 as qr
dev = torch.device("cuda:0"); st = torch.cuda.current_stream()
def t(fn, reps=5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
n, m, L = 1 << 26, 10**6, 32
text = torch.empty((n + 31) // 32 + 1, dtype=torch.uint64, device=dev); gen.dna_dev(4, n, 0, text)
fm = qr.qr_fm_build(text, n)
pats = torch.empty(m * L, dtype=torch.uint8, device=dev); gen.patterns_dev(4, 0, m, L, text, n, pats)
out = torch.empty(m, dtype=torch.int32, device=dev)
for dyn in (0, 1):
    qr.qr_set_tuning("fm_dyn", dyn)
    ms = t(lambda: qr.qr_fm_count_approx(fm, pats, None, L, 1, out, m, st))
    print(json.dumps({"approx1": "c4", "dyn": dyn, "ms": ms, "gpat_s": m / ms / 1e6, "checksum": int(out.to(torch.int64).sum())}), flush=True)
PY
timeout 600 python /tmp/approx_probe.py > gpurun_out/approx_probe.jsonl 2>&1
