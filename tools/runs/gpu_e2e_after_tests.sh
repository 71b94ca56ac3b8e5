cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
(cat /proc/buddyinfo; grep -E "MemFree|AnonHuge|Cached" /proc/meminfo) > gpurun_out/host_before.txt
timeout 600 python tools/e2e_host_probe.py > gpurun_out/e2e_fresh.jsonl 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 -x > gpurun_out/pytest_gpu.log 2>&1
(cat /proc/buddyinfo; grep -E "MemFree|AnonHuge|Cached" /proc/meminfo; ps aux --sort=-%cpu | head -15) > gpurun_out/host_after.txt
timeout 600 python tools/e2e_host_probe.py > gpurun_out/e2e_after.jsonl 2>&1
sync; echo 3 > /proc/sys/vm/drop_caches 2>/dev/null; echo 1 > /proc/sys/vm/compact_memory 2>/dev/null
(cat /proc/buddyinfo; grep -E "MemFree|AnonHuge|Cached" /proc/meminfo) > gpurun_out/host_compacted.txt
timeout 600 python tools/e2e_host_probe.py > gpurun_out/e2e_compacted.jsonl 2>&1
