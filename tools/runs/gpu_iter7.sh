cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fm.py -q --timeout 900 -x -rf > gpurun_out/pytest_fm.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fm.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --rows headline --dist-backend gloo > gpurun_out/bench_2rank.log 2>&1
echo "2rank exit $?" >> gpurun_out/bench_2rank.log
