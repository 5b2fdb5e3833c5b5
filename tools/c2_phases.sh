timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1
timeout 600 python bench.py --no-extras --no-cpu-baseline --ttft 1200 > gpurun_out/bench_c2lx.json 2>&1
timeout 600 python bench.py --only c5x --no-cpu-baseline --c5x-decisions 1024 > gpurun_out/bench_c5x.json 2>&1
