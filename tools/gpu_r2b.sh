# Exhaustive MPC change check: parity suites, then C2 (tight and loose SLO) and C5 exhaustive timings.
set -x
timeout 900 python -m pytest tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_exhaustive_deep.py -x -q > gpurun_out/pytest_b.log 2>&1; echo pytest=$?
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 600 python bench.py --only c2l --no-cpu-baseline > gpurun_out/bench_c2l.json 2> gpurun_out/bench_c2l.err; echo c2l=$?
timeout 600 python bench.py --only c5x --no-cpu-baseline > gpurun_out/bench_c5x.json 2> gpurun_out/bench_c5x.err; echo c5x=$?
