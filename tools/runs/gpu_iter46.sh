cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fm.py -q --timeout 1200 -x -rf -k "quadrank16x2" > gpurun_out/pytest_fm.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fm.log
timeout 900 python tools/fm_layout_probe.py > gpurun_out/fm_layout.jsonl 2>&1
