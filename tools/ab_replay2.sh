# C4 replay and the C1 scenario: default library vs a variant, alternating; replay parity tests
for v in base $1 base $1; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])['c4_replay']; print('$v c4', round(d['value']))"
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])['c1_demo']; print('$v c1', round(d['value']), d.get('phase_ms'), round(d['replicas']['value']))"
done
timeout 900 python -m pytest -q -m gpu tests/test_gpu_replay.py tests/test_gpu_daysim.py -x 2>&1 | tail -1
