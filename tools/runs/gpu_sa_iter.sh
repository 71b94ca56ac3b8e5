cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fm.py -q --timeout 900 -x -rf > gpurun_out/pytest_fm.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fm.log
timeout 900 python tools/fm_build_probe.py > gpurun_out/fm_build_probe.jsonl 2>&1
echo "probe exit $?" >> gpurun_out/fm_build_probe.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/build_launches.csv python tools/fm_build_probe.py once > gpurun_out/build_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/build_ncu.log
