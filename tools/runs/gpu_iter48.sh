cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 600 python bench.py --rows headline --no-cpu > gpurun_out/bench_head.jsonl 2>&1
echo "exit $?" >> gpurun_out/bench_head.jsonl
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --rows headline --no-cpu --dist-backend gloo > gpurun_out/bench_2rank.log 2>&1
echo "2rank exit $?" >> gpurun_out/bench_2rank.log
