cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
timeout 300 python tools/fm_l1_driver.py > gpurun_out/fm_l1_plain.log 2>&1 && \
timeout 900 ncu --clock-control none -k regex:k_fm_count -c 2 --csv --metrics \
gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_lg.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_global_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed.sum,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct \
python tools/fm_l1_driver.py > gpurun_out/fm_l1_ncu.csv 2>&1
echo "exit $?" >> gpurun_out/fm_l1_ncu.csv
