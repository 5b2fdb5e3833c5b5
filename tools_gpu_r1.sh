# round-1 GPU measurement recipe (run from the repo root under gpurun)
set -x
for D in 256 1024 4096; do
  python bench.py --no-extras --no-cpu-baseline --steps 10 --decisions $D > gpurun_out/c2_d$D.json 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv \
    python bench.py --no-extras --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/c2_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/sweep_full \
    python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/sweep_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv \
    python bench.py --only c3 --no-cpu-baseline > gpurun_out/c3_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:probe_kernel -c 1 -o gpurun_out/probe_full \
    python bench.py --only c3 --no-cpu-baseline > gpurun_out/probe_full.log 2>&1
