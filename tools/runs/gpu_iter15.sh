cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_fm.py -q --timeout 1200 -x -rf > gpurun_out/pytest_fm2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fm2.log
