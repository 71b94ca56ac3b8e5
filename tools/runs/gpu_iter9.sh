cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_rank.py -q --timeout 900 -x -rf > gpurun_out/pytest_var.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_var.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
