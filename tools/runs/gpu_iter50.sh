cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_variants.py -q --timeout 1200 -x -rf > gpurun_out/pytest_var.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_var.log
timeout 1200 python tools/size_sweep.py bits_only > gpurun_out/size_sweep_b32.jsonl 2>&1
