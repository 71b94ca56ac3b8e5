cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -q --timeout 600 -x -rf > gpurun_out/pytest_mr.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_mr.log
timeout 300 python tools/profile_driver.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_(bi_rank2|bi_gather2|qd_rank2|qd_all4_2|b64_rank|q64_rank|fm_count|fm_approx1)' -c 12 -o gpurun_out/prof_r01_final -f \
  python tools/profile_driver.py > gpurun_out/ncu_final.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_final.log
timeout 600 python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launches.log
