cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_fm.py -q --timeout 1200 -x -rf -k "16x2 or chain or save_load" > gpurun_out/pytest_q16.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_q16.log
timeout 1200 python tools/size_sweep.py dna_only > gpurun_out/size_sweep_q16x2b.jsonl 2>&1
timeout 900 python tools/fm_layout_probe.py > gpurun_out/fm_layout2.jsonl 2>&1
