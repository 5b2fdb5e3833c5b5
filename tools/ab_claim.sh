bash tools/ab_variant.sh cl32 | sed 's/^var/cl32/'
bash tools/ab_variant.sh cl256 | grep "^var" | sed 's/^var/cl256/'
for v in base c3x64 c3x512 base; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c5x --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c5x', round(d['c5_exhaustive']['value']))"
done
