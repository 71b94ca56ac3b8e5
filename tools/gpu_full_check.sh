cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 -x -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
