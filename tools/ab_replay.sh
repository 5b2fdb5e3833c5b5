# C4 replay (1024 scenarios) and the C1 single scenario with replay register-budget variants
for v in base "$@" base; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])['c4_replay']; print('$v c4', round(d['value']), d.get('phase_ms'))"
  env ${L:+BS_LIB_PATH=$L} timeout 600 python tools/c1_replay.py > /dev/null 2>&1
done
