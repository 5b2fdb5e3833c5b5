python tools/c1_latency.py
BS_LIB_PATH=$PWD/paper_2602_18755_b200/libbiscale_gpu_gph.so python tools/c1_latency.py > gpurun_out/c1gph.log 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_replay.py -x 2>&1 | tail -1
