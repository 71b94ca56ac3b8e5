# headline launch list + full ncu capture of every hot kernel (run under gpurun from the repo root)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 600 python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
timeout 300 python tools/profile_driver.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_(bi_rank|bi_gather|qd_rank|qd_all4|fm_count|b64|q64|fm_approx)' -c 20 -o gpurun_out/prof_final -f \
  python tools/profile_driver.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
