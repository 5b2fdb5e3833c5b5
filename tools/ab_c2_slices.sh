# A/B of C2 e2e: default build ("new": one pack slice at 1024 problems) vs libbiscale_gpu_sl256.so ("old" label: 4 slices of 256).
V=$PWD/paper_2602_18755_b200/libbiscale_gpu_sl256.so
for i in 1 2 3 4; do
  timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ab_new$i.json 2>/dev/null
  BS_LIB_PATH=$V timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ab_old$i.json 2>/dev/null
done
python - <<'PY'
import json, statistics
for tag in ("new","old"):
    v=[];e=[]
    for i in range(1,5):
        d=json.loads([l for l in open(f"gpurun_out/ab_{tag}{i}.json") if l.startswith("{")][0]); v.append(d["value"]); e.append(d["e2e"]["value"])
    print(tag, "value", ["%.3e"%x for x in v], "e2e", ["%.3e"%x for x in e], "median e2e %.3e"%statistics.median(e))
PY
