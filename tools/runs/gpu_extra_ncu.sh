cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 300 python tools/extra_driver.py > gpurun_out/extra_plain.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:k_bi_rank1s|k_fm_approx1' -c 2 -o /tmp/extra -f python tools/extra_driver.py > gpurun_out/extra_ncu.log 2>&1
echo "exit $?" >> gpurun_out/extra_ncu.log
python tools/ncu_summary.py /tmp/extra.ncu-rep > gpurun_out/extra_summary.md 2>&1
ncu -i /tmp/extra.ncu-rep --page raw --csv > gpurun_out/extra_raw.csv 2>/dev/null
