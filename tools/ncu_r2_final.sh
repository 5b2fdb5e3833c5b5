bash tools/ncu_sweep.sh
M=gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio,launch__registers_per_thread,launch__grid_size,launch__block_size
timeout 1500 ncu --metrics $M --clock-control none -k "regex:sweep_kernel" -s 3 -c 1 --csv --log-file gpurun_out/roof_c2l.csv python bench.py --only c2l --no-cpu-baseline > gpurun_out/roof_c2l.log 2>&1
timeout 1500 ncu --metrics $M --clock-control none -k "regex:greedy" -s 2 -c 1 --csv --log-file gpurun_out/roof_c5g.csv python bench.py --only c5g --no-cpu-baseline > gpurun_out/roof_c5g.log 2>&1
for i in 1 2 3; do timeout 600 python bench.py --only c5g --no-cpu-baseline > gpurun_out/c5g_$i.json 2>/dev/null; done
