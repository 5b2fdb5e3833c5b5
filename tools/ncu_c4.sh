# ncu source profile of the C4 replay's prefill kernel (1024 scenarios)
timeout 600 python bench.py --only c4 --no-cpu-baseline > gpurun_out/c4_pre.json 2>&1; echo pre=$?
ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 1 -c 1 -o gpurun_out/c4p_full python bench.py --only c4 --no-cpu-baseline > gpurun_out/c4p_full.log 2>&1; echo ncu=$?
