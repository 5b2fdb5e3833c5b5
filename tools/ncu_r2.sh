# ncu captures of the exhaustive-MPC kernels at C2 (1024 decisions), after the same command ran clean.
set -x
F="ncu --set full --clock-control none --import-source on"
timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_pre.json 2>&1; echo pre=$?
$F -k regex:thr_kernel -s 2 -c 1 -o gpurun_out/thr_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/thr_full.log 2>&1
$F -k regex:bfs_node_kernel -s 2 -c 1 -o gpurun_out/bfs_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/bfs_full.log 2>&1
$F -k regex:sweep_kernel -s 2 -c 1 -o gpurun_out/sweep_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/sweep_full.log 2>&1
ls -la gpurun_out
