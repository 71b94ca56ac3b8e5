# headline launch list + full ncu capture of every hot kernel (run under gpurun from the repo root);
# the .ncu-rep is summarised on the box and deleted (gpurun brings back <= 64 MiB)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 600 python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
timeout 300 python tools/profile_driver.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_(bi_rank|bi_gather|qd_rank|qd_all4|fm_count|b64|q64|fm_approx|b16x2|q16x2)' -c 26 -o /tmp/prof_final -f \
  python tools/profile_driver.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
python tools/ncu_summary.py /tmp/prof_final.ncu-rep > gpurun_out/prof_final_summary.md 2>&1
ncu -i /tmp/prof_final.ncu-rep --page raw --csv > gpurun_out/prof_final_raw.csv 2>/dev/null
ncu -i /tmp/prof_final.ncu-rep --page details --csv > gpurun_out/prof_final_details.csv 2>/dev/null
ls -la gpurun_out >> gpurun_out/ncu_full.log
