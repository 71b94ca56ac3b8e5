# tests + sweep + bench (run under gpurun from the repo root)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -x -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/grid_sweep.py > gpurun_out/grid.jsonl 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
