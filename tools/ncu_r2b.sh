set -x
timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_pre.json 2>&1; echo pre=$?
ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,smsp__warps_launched.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/c2_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:thr_kernel -s 2 -c 1 -o gpurun_out/thr_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/thr_full.log 2>&1
