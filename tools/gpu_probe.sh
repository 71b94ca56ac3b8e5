cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/gather_probe 2147483648 100000000 > gpurun_out/probe.jsonl 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_op_read_hit_rate.pct \
  --clock-control none --csv --log-file gpurun_out/probe_ncu.csv ./tools/gather_probe 2147483648 100000000 > gpurun_out/probe_ncu.log 2>&1
echo "probe exit $?" >> gpurun_out/probe.jsonl
timeout 600 python tools/grid_sweep.py > gpurun_out/grid.jsonl 2>&1
