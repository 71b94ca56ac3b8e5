cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 -x -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/fm_build_probe.py > gpurun_out/fm_build_probe.jsonl 2>&1
echo "probe exit $?" >> gpurun_out/fm_build_probe.jsonl
