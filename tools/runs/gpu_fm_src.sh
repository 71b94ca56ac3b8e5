cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fm_count -c 2 -o /tmp/fm_src -f \
  python tools/fm_l1_driver.py > gpurun_out/fm_src_ncu.log 2>&1
echo "exit $?" >> gpurun_out/fm_src_ncu.log
ncu -i /tmp/fm_src.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/fm_src_source.csv 2>gpurun_out/fm_src_err.log
ncu -i /tmp/fm_src.ncu-rep --page raw --csv > gpurun_out/fm_src_raw.csv 2>>gpurun_out/fm_src_err.log
ls -la gpurun_out/fm_src_* >> gpurun_out/fm_src_ncu.log
