cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
for i in 1 2; do
timeout 600 python bench.py --rows headline --no-cpu > gpurun_out/bench_new_$i.jsonl 2>&1
timeout 600 python bench_prev.py --rows headline --no-cpu > gpurun_out/bench_prev_$i.jsonl 2>&1
done
