# A/B of a compile-time variant against the default library on the C2 headline:
# tools/ab_variant.sh NAME [extra bench args]
V=$PWD/paper_2602_18755_b200/libbiscale_gpu_$1.so; shift
for i in 1 2 3; do
  timeout 600 python bench.py --no-extras --no-cpu-baseline "$@" > gpurun_out/ab_base$i.json 2>/dev/null
  BS_LIB_PATH=$V timeout 600 python bench.py --no-extras --no-cpu-baseline "$@" > gpurun_out/ab_var$i.json 2>/dev/null
done
python - <<'PY'
import json
for tag in ("base", "var"):
    for i in (1, 2, 3):
        d = json.loads(open(f"gpurun_out/ab_{tag}{i}.json").read().strip().splitlines()[-1])
        print(tag, i, f"{d['value']:.4g}", f"{d['ms_per_step']:.4f}", {k: round(v, 4) for k, v in d['phase_ms_avg'].items()})
PY
