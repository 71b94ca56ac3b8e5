cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1300 python tools/size_sweep.py > gpurun_out/size_sweep3.jsonl 2>&1
