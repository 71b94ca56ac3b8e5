cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu > gpurun_out/tma_build.log 2>&1
timeout 300 ./tools/tma_probe 2147483648 200000000 > gpurun_out/tma_probe.jsonl 2>&1
echo "exit $?" >> gpurun_out/tma_probe.jsonl
