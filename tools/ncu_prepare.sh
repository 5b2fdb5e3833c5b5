set -x
timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_pre.json 2>&1; echo pre=$?
ncu --set full --clock-control none --import-source on -k regex:prepare_kernel -s 2 -c 1 -o gpurun_out/prep_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/prep_full.log 2>&1
