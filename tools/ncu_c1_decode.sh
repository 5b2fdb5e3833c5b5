# ncu source profile of the C1 scenario's decode_kernel (one scenario, one warp)
timeout 300 python tools/c1_replay.py > gpurun_out/c1r_pre.log 2>&1; echo pre=$?
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 -o gpurun_out/c1dec_full python tools/c1_replay.py > gpurun_out/c1dec_full.log 2>&1; echo ncu=$?
