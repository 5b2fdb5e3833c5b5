# Round-1 GPU measurement recipe (run from the repo root under gpurun).
# Every ncu command runs only after the same command exited 0 without ncu.
set -x
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches_d1024.csv \
    python bench.py --no-extras --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/c2_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/sweep_full_d1024 \
    python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/sweep_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv \
    python bench.py --only c4 --no-cpu-baseline > gpurun_out/c4_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"prefill_kernel|decode_kernel" -c 2 -o gpurun_out/replay_full3 \
    python bench.py --only c4 --no-cpu-baseline --c4-scenarios 256 > gpurun_out/replay_full3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv \
    python bench.py --only c5g --no-cpu-baseline > gpurun_out/c5_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -c 1 -o gpurun_out/greedy_full \
    python bench.py --only c5g --no-cpu-baseline > gpurun_out/greedy_full.log 2>&1
