cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 300 python tools/profile_smem.py > gpurun_out/prof_smem_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_(bi_rank2|qd_rank2|qd_all4_2)' -c 6 -o gpurun_out/prof_smem -f \
  python tools/profile_smem.py > gpurun_out/ncu_smem.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_smem.log
