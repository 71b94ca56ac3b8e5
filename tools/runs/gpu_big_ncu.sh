cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 600 python tools/big_driver.py > gpurun_out/big_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none -k 'regex:k_bi_rank2v|k_qd_rank2w' -c 2 -o /tmp/big -f python tools/big_driver.py > gpurun_out/big_ncu.log 2>&1
echo "exit $?" >> gpurun_out/big_ncu.log
python tools/ncu_summary.py /tmp/big.ncu-rep > gpurun_out/big_summary.md 2>&1
