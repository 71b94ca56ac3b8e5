cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 300 python tools/small_driver.py > gpurun_out/small_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bi_rank -c 2 -o /tmp/small -f python tools/small_driver.py > gpurun_out/small_ncu.log 2>&1
echo "exit $?" >> gpurun_out/small_ncu.log
python tools/ncu_summary.py /tmp/small.ncu-rep > gpurun_out/small_summary.md 2>&1
ncu -i /tmp/small.ncu-rep --page raw --csv > gpurun_out/small_raw.csv 2>/dev/null
