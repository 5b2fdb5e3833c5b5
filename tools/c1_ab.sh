# Controller-call latency with and without the cluster launch, then the greedy parity tests.
for i in 1 2; do
  python tools/c1_latency.py | sed 's/^/cluster /'
  BS_GREEDY_NO_CLUSTER=1 python tools/c1_latency.py | sed 's/^/cta /'
done
timeout 900 python -m pytest -q -m gpu tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_replay.py -x 2>&1 | tail -2
