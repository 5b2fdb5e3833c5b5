# Greedy MPC (multi-warp decisions for small batches): parity, per-call latency, C5 greedy, C1.
set -x
timeout 900 python -m pytest tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_exhaustive_deep.py tests/test_gpu_cluster_replay.py -x -q > gpurun_out/pytest_d.log 2>&1; echo pytest=$?
python tools/c1_latency.py > gpurun_out/c1lat.txt 2>&1
BS_DEBUG_TIMING=1 python tools/c1_latency.py 2>&1 | tail -3 > gpurun_out/c1lat_dbg.txt
timeout 600 python bench.py --only c5g --no-cpu-baseline > gpurun_out/bench_c5g.json 2>&1; echo c5g=$?
timeout 600 python bench.py --only c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>&1; echo c1=$?
