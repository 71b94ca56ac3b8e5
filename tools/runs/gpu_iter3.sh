cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 600 python tools/s_probe.py > gpurun_out/s_probe.jsonl 2>&1
timeout 300 python tools/s_probe.py once > gpurun_out/s_once.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_bi_(rank2|gather2)' -c 4 -o gpurun_out/prof_pair -f python tools/s_probe.py once > gpurun_out/ncu_pair.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_pair.log
