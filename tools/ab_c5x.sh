# C5 exhaustive (24^8): default library vs a variant, alternating, then the deep parity tests
for v in base $1 base $1; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c5x --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c5x', round(d['c5_exhaustive']['value']))"
done
timeout 900 python -m pytest tests/test_gpu_exhaustive_deep.py tests/test_golden.py -x -q 2>&1 | tail -1
