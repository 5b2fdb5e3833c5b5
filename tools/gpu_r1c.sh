# Round-1 final measurement of the current code (run from the repo root under gpurun):
# the GPU suite, the default bench line, then (each after its command exited 0 without ncu)
# launch lists and full captures of the dominant kernels.
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
L="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
F="ncu --set full --clock-control none --import-source on"
$L --log-file gpurun_out/c2_launches.csv python bench.py --no-extras --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/c2_launches.log 2>&1
$F -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/sweep_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/sweep_full.log 2>&1
$F -k regex:bfs_node_kernel -s 6 -c 2 -o gpurun_out/bfs_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/bfs_full.log 2>&1
$F -k regex:prepare_kernel -s 3 -c 1 -o gpurun_out/prepare_full python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/prepare_full.log 2>&1
$L --log-file gpurun_out/c3_launches.csv python bench.py --only c3 --no-cpu-baseline > gpurun_out/c3_launches.log 2>&1
$L --log-file gpurun_out/c5x_launches.csv python bench.py --only c5x --no-cpu-baseline --c5x-decisions 1024 > gpurun_out/c5x_launches.log 2>&1
$F -k regex:probe_kernel -c 1 -o gpurun_out/probe_full python bench.py --only c3 --no-cpu-baseline > gpurun_out/probe_full.log 2>&1
ls -la gpurun_out
