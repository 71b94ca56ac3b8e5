#!/bin/bash
# Round evidence on one B200 (under gpurun, repo root): build, the GPU test suite, smoke, the
# driver's bench command, the ncu launch list of the headline bench and ncu --set full of every
# hot kernel (tools/profile_driver.py), summarised on the box (the .ncu-rep is not copied back).
# TAG names the files (default r02f).
set -u
TAG=${TAG:-r02f}
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out
mkdir -p $O
make -s all > $O/${TAG}_make.log 2>&1
nvidia-smi --query-gpu=serial,name,driver_version --format=csv,noheader > $O/${TAG}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -x -rf > $O/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/${TAG}_bench.jsonl 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > /dev/null 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv \
      python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > $O/${TAG}_launches.log 2>&1
python tools/profile_driver.py > /dev/null 2>&1 && \
  timeout 1500 ncu --set full --clock-control none -k regex:"k_bi_rank2c|k_qd_rank2c|k_qd_all4_2c|k_fm_count|k_fm_seed|k_fm_approx|k_ax_" \
      -o $O/${TAG}_full python tools/profile_driver.py > $O/${TAG}_ncu.log 2>&1
if [ -f $O/${TAG}_full.ncu-rep ]; then
  ncu -i $O/${TAG}_full.ncu-rep --page raw --csv > $O/${TAG}_ncu_raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/${TAG}_full.ncu-rep > $O/${TAG}_ncu_summary.md 2>&1
  python tools/ncu_traffic.py $O/${TAG}_full.ncu-rep profiles/${TAG}_ncu.md "$(cut -d, -f1 $O/${TAG}_gpu.txt)" \
      > $O/${TAG}_traffic.log 2>&1; cp profiles/traffic.json $O/${TAG}_traffic.json
  rm -f $O/${TAG}_full.ncu-rep
fi
ls -la $O | grep $TAG
