cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_rank.py -q --timeout 900 -x -rf > gpurun_out/pytest_rank.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_rank.log
timeout 600 python tools/e2e_sweep.py > gpurun_out/e2e_sweep.jsonl 2>&1
timeout 600 compute-sanitizer --tool memcheck --leak-check no python __graft_entry__.py smoke > gpurun_out/memcheck.log 2>&1
echo "memcheck exit $?" >> gpurun_out/memcheck.log
