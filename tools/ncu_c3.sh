# ncu full capture of the C3 probe kernel (one table stream launch)
timeout 600 python bench.py --only c3 --no-cpu-baseline > gpurun_out/c3_pre.json 2>&1; echo pre=$?
ncu --set full --clock-control none --import-source on -k regex:probe_kernel -s 1 -c 1 -o gpurun_out/c3p_full python bench.py --only c3 --no-cpu-baseline > gpurun_out/c3p_full.log 2>&1; echo ncu=$?
