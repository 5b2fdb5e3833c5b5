timeout 900 python -m pytest tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_exhaustive_deep.py -x -q > gpurun_out/pytest_x.log 2>&1; echo pytest=$?
for i in 1 2; do timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_x$i.json 2> gpurun_out/bench_x.err; done
timeout 600 python bench.py --only c2l --no-cpu-baseline > gpurun_out/bench_x_c2l.json 2>> gpurun_out/bench_x.err
timeout 600 python bench.py --only c5x --no-cpu-baseline > gpurun_out/bench_x_c5x.json 2>> gpurun_out/bench_x.err
