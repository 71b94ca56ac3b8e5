cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_rank.py tests/test_gpu_fullsize.py -q --timeout 900 -x -rf -k "quadrank or config3 or index64" > gpurun_out/pytest_qd.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_qd.log
SWEEP_K=1,2,4 SWEEP_BPS=32,64 SWEEP_PAIR=1 timeout 900 python tools/grid_sweep.py > gpurun_out/grid3.jsonl 2>&1
