cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_rank.py -q --timeout 1200 -rf > gpurun_out/pytest_fuzz.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fuzz.log
