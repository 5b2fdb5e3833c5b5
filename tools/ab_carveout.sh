bash tools/ab_variant.sh co0
bash tools/ab_variant.sh co100 | grep "^var" | sed 's/^var/co100/'
for v in base co0; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c5x --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c5x', round(d['c5_exhaustive']['value']))"
done
