# ncu source profile of the C5 (24^8) three-level sweep
timeout 600 python bench.py --only c5x --no-cpu-baseline > gpurun_out/c5x_pre.json 2>&1; echo pre=$?
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o gpurun_out/c5x_full python bench.py --only c5x --no-cpu-baseline > gpurun_out/c5x_full.log 2>&1; echo ncu=$?
