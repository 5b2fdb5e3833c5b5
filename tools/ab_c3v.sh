for v in "$@"; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} timeout 300 python tools/decode_probe_profile.py 2>&1 | tail -1 | sed "s/^/$v /"
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])['c3_placement']; print('$v', round(d['value']), round(d['table_s'],3), round(d['phase_ms']['probe'],1))"
done
