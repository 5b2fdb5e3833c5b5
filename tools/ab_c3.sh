# C3 table stream and the longest probe with compile-time variants: tools/ab_c3.sh VARIANT...
for v in base "$@"; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  for i in 1 2; do
    env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c3 --no-cpu-baseline > gpurun_out/c3_$v$i.json 2>/dev/null
  done
  env ${L:+BS_LIB_PATH=$L} timeout 300 python tools/decode_probe_profile.py > gpurun_out/dpp_$v.log 2>&1
done
python - "$@" <<'PY'
import json, sys
for v in ["base"] + sys.argv[1:]:
    for i in (1, 2):
        d = json.loads(open(f"gpurun_out/c3_{v}{i}.json").read().strip().splitlines()[-1])["c3_placement"]
        print(v, i, round(d["value"]), round(d["table_s"], 3), d["phase_ms"])
    print(v, open(f"gpurun_out/dpp_{v}.log").read().strip().splitlines()[-1])
PY
