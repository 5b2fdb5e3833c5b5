# Executed-roofline metrics of each sub-benchmark's dominant kernel (one
# launch each, after warm-up) -> gpurun_out/roof_<cfg>.csv; summarised into
# profiles/r02_rooflines.json by tools/rooflines_json.py.
set -x
M=gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed_per_inst_executed.ratio,launch__registers_per_thread,launch__grid_size,launch__block_size
run() {  # cfg kernel-regex skip
  timeout 1500 ncu --metrics $M --clock-control none -k "regex:$2" -s $3 -c 1 --csv --log-file gpurun_out/roof_$1.csv \
    python bench.py --only $1 --no-cpu-baseline > gpurun_out/roof_$1.log 2>&1; echo $1=$?
}
run c1 decode_kernel 1
run c2l sweep_kernel 3
run c3 probe_kernel 1
run c4 prefill_kernel 1
run c4d "prefill_kernel|probe_kernel" 1
run c4x probe_kernel 1
run c5g greedy 2
run c5x sweep_kernel 2
