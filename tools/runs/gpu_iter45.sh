cd $GRAFT_REPO_ROOT
bash tools/gpu_full_check.sh
timeout 1200 python tools/size_sweep.py dna_only > gpurun_out/size_sweep_q16x2.jsonl 2>&1
