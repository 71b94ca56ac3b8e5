cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fm.py -q --timeout 1200 -x -rf -k "approx" > gpurun_out/pytest_fm.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fm.log
timeout 300 python tools/approx_probe.py k > gpurun_out/approx_probe.jsonl 2>&1
echo "probe exit $?" >> gpurun_out/approx_probe.jsonl
