# C5 greedy, C1 controller call and C4 replay: default library vs a variant; greedy parity tests
for v in base $1 base $1; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c5g --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c5g', round(d['c5_greedy']['value']))"
  env ${L:+BS_LIB_PATH=$L} python tools/c1_latency.py | sed "s/^/$v /"
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])['c4_replay']; print('$v c4', round(d['value']))"
done
timeout 900 python -m pytest -q -m gpu tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_replay.py -x 2>&1 | tail -1
