# ncu --set full of the C2 sweep (the bench's dominant kernel) after the same command ran clean,
# plus the launch list of one C2 step.
set -x
timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_pre.json 2>&1; echo pre=$?
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o gpurun_out/sweep_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/sweep_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --no-extras --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/c2_launches.log 2>&1
