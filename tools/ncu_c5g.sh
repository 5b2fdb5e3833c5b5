# ncu source profile of the C5 greedy batch kernel
timeout 600 python bench.py --only c5g --no-cpu-baseline > gpurun_out/c5g_pre.json 2>&1; echo pre=$?
ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -s 2 -c 1 -o gpurun_out/c5g_full python bench.py --only c5g --no-cpu-baseline > gpurun_out/c5g_full.log 2>&1; echo ncu=$?
