cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_rank.py -k "index64" -q --timeout 900 -x -rf > gpurun_out/pytest_idx.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_idx.log
timeout 900 python tools/fm_sweep.py > gpurun_out/fm_sweep.jsonl 2>&1
