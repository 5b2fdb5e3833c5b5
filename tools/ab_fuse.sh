# A/B of the BFS fusion of dominated depth-(K-2) nodes: default build vs libbiscale_gpu_nofuse.so (sweep-only node tests).
V=$PWD/paper_2602_18755_b200/libbiscale_gpu_nofuse.so
for i in 1 2; do
  timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ab_fuse_c2_new$i.json 2>/dev/null
  BS_LIB_PATH=$V timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/ab_fuse_c2_old$i.json 2>/dev/null
  timeout 300 python bench.py --only c2l --no-cpu-baseline > gpurun_out/ab_fuse_c2l_new$i.json 2>/dev/null
  BS_LIB_PATH=$V timeout 300 python bench.py --only c2l --no-cpu-baseline > gpurun_out/ab_fuse_c2l_old$i.json 2>/dev/null
done
BS_LIB_PATH=$V timeout 300 python bench.py --only c5x --no-cpu-baseline > gpurun_out/ab_fuse_c5x_old.json 2>/dev/null
python - <<'PY'
import json
def ld(f): return json.loads([l for l in open(f) if l.startswith("{")][-1])
for tag in ("new", "old"):
    for i in (1, 2):
        a = ld(f"gpurun_out/ab_fuse_c2_{tag}{i}.json"); b = ld(f"gpurun_out/ab_fuse_c2l_{tag}{i}.json")["c2_loose_slo"]
        print(tag, i, "c2 step %.4f" % a["ms_per_step"], {k: round(v, 4) for k, v in a["phase_ms_avg"].items()},
              "c2l step %.3f sweep %.3f" % (b["ms_per_step"], b["sweep_ms"]))
print("c5x nofuse", ld("gpurun_out/ab_fuse_c5x_old.json")["c5_exhaustive"]["value"])
PY
