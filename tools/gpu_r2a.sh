# Round 2: parity of the new paths, then the default bench line.
set -x
timeout 900 python -m pytest tests/test_gpu_placement.py tests/test_golden.py tests/test_gpu_exhaustive_deep.py -x -q > gpurun_out/pytest_a.log 2>&1; echo pytest=$?
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
