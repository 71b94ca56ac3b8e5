cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and not slow" -q --timeout 400 -x -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
SWEEP_K=2,4,8 SWEEP_BPS=8,16,32,64 timeout 900 python tools/grid_sweep.py > gpurun_out/grid2.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q --timeout 900 -rf > gpurun_out/pytest_full.log 2>&1
echo "pytest full exit $?" >> gpurun_out/pytest_full.log
