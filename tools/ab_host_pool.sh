# A/B of the host-pool width: default build vs libbiscale_gpu_w7.so (7 workers, grains 128), same box.
V=$PWD/paper_2602_18755_b200/libbiscale_gpu_w7.so
nproc
for i in 1 2 3 4; do
  timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ab_new$i.json 2>/dev/null
  BS_LIB_PATH=$V timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ab_old$i.json 2>/dev/null
done
for i in 1 2; do
  timeout 300 python bench.py --only c5g --no-cpu-baseline > gpurun_out/ab_c5g_new$i.json 2>/dev/null
  BS_LIB_PATH=$V timeout 300 python bench.py --only c5g --no-cpu-baseline > gpurun_out/ab_c5g_old$i.json 2>/dev/null
done
python - <<'PY'
import json, statistics
def ld(f): return json.loads([l for l in open(f) if l.startswith("{")][0])
for tag, name in (("new", "default"), ("old", "w7")):
    e = [ld(f"gpurun_out/ab_{tag}{i}.json")["e2e"]["value"] for i in range(1, 5)]
    v = [ld(f"gpurun_out/ab_{tag}{i}.json")["value"] for i in range(1, 5)]
    g = [ld(f"gpurun_out/ab_c5g_{tag}{i}.json")["c5_greedy"]["value"] for i in (1, 2)]
    print(name, "value %.3e" % statistics.median(v), "e2e", ["%.3e" % x for x in e], "median %.3e" % statistics.median(e),
          "c5g", ["%.3e" % x for x in g])
PY
