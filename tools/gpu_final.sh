#!/bin/bash
# Round-2 evidence run on one B200 (under gpurun): the driver's bench command, the ncu launch
# list of the headline bench, and ncu --set full of every hot kernel (tools/profile_driver.py),
# summarised on the box (the .ncu-rep files are deleted: gpurun copies back <= 64 MiB).
set -u
O=gpurun_out
nvidia-smi --query-gpu=serial,name,driver_version --format=csv,noheader > $O/r02_gpu.txt
python bench.py --steps 20 --warmup 5 > $O/r02_bench_final.jsonl 2> $O/r02_bench_final.err
python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches.csv \
      python bench.py --rows headline --no-cpu --steps 2 --warmup 3 > $O/r02_launches.log 2>&1
python tools/profile_driver.py > /dev/null 2>&1 && \
  ncu --set full --clock-control none -k regex:"k_bi_rank2c|k_qd_rank2c|k_qd_all4_2c|k_fm_count|k_fm_seed|k_fm_approx" \
      -o $O/r02_final python tools/profile_driver.py > $O/r02_ncu_final.log 2>&1
if [ -f $O/r02_final.ncu-rep ]; then
  ncu -i $O/r02_final.ncu-rep --page raw --csv > $O/r02_ncu_final_raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/r02_final.ncu-rep > $O/r02_ncu_final_summary.md 2>&1
  python tools/ncu_traffic.py $O/r02_final.ncu-rep profiles/r02_ncu_final.md "$(cut -d, -f1 $O/r02_gpu.txt)" \
      > $O/r02_traffic.log 2>&1; cp profiles/traffic.json $O/r02_traffic.json
  rm -f $O/r02_final.ncu-rep
fi
ls -la $O
