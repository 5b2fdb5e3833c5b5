# Round-1 profile refresh of the current kernels (run from the repo root under gpurun).
# Every ncu command runs only after the same command exited 0 without ncu (bench_default.json).
set -x
L="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
F="ncu --set full --clock-control none --import-source on"
$L --log-file gpurun_out/c2_launches.csv python bench.py --no-extras --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/c2_launches.log 2>&1
$F -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/sweep_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/sweep_full.log 2>&1
$F -k regex:bfs_kernel -s 14 -c 4 -o gpurun_out/bfs_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/bfs_full.log 2>&1
$L --log-file gpurun_out/c1_launches.csv python bench.py --only c1 --no-cpu-baseline > gpurun_out/c1_launches.log 2>&1
$L --log-file gpurun_out/c3_launches.csv python bench.py --only c3 --no-cpu-baseline > gpurun_out/c3_launches.log 2>&1
$L --log-file gpurun_out/c4_launches.csv python bench.py --only c4 --no-cpu-baseline > gpurun_out/c4_launches.log 2>&1
$L --log-file gpurun_out/c5g_launches.csv python bench.py --only c5g --no-cpu-baseline > gpurun_out/c5g_launches.log 2>&1
$L --log-file gpurun_out/c5x_launches.csv python bench.py --only c5x --no-cpu-baseline --c5x-decisions 1024 > gpurun_out/c5x_launches.log 2>&1
$F -k regex:probe_kernel -c 1 -o gpurun_out/probe_full python bench.py --only c3 --no-cpu-baseline > gpurun_out/probe_full.log 2>&1
$F -k regex:"decode_kernel|prefill_kernel" -c 2 -o gpurun_out/c1_replay_full python bench.py --only c1 --no-cpu-baseline > gpurun_out/c1_replay_full.log 2>&1
ls -la gpurun_out
