# Exhaustive MPC: parity, C2 / C2-loose / C5x timings, then the sweep work counters (BS_SWEEP_STATS build).
set -x
timeout 900 python -m pytest tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_exhaustive_deep.py -x -q > gpurun_out/pytest_c.log 2>&1; echo pytest=$?
timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 600 python bench.py --only c2l --no-cpu-baseline > gpurun_out/bench_c2l.json 2> gpurun_out/bench_c2l.err; echo c2l=$?
timeout 600 python bench.py --only c5x --no-cpu-baseline > gpurun_out/bench_c5x.json 2> gpurun_out/bench_c5x.err; echo c5x=$?
V=$PWD/paper_2602_18755_b200/libbiscale_gpu_stats.so
BS_LIB_PATH=$V BS_DEBUG_COUNTS=1 timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2> gpurun_out/stats_c2.err
BS_LIB_PATH=$V BS_DEBUG_COUNTS=1 timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 1 --warmup 3 --ttft 1200 > /dev/null 2> gpurun_out/stats_c2l.err
timeout 600 python bench.py --no-extras --no-cpu-baseline --ttft 1200 > gpurun_out/bench_c2lx.json 2>&1; echo c2lx=$?
