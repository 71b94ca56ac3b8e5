cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 900 python tools/smem_probe.py > gpurun_out/smem_probe2.jsonl 2>&1
echo "probe exit $?" >> gpurun_out/smem_probe2.jsonl
