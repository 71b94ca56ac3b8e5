cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sbcache.py tests/test_gpu_rank.py -q --timeout 1200 -x -rf > gpurun_out/pytest_rank.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_rank.log
timeout 1300 python tools/regime_probe.py > gpurun_out/regime2.jsonl 2>&1
