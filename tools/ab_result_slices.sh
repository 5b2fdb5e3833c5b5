# A/B of the sliced result copy-back (expansion of a slice overlaps the next slice's D2H) vs libbiscale_gpu_r1.so (one slice).
V=$PWD/paper_2602_18755_b200/libbiscale_gpu_r1.so
timeout 600 python -m pytest tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_experiment.py tests/test_gpu_cluster_replay.py -m gpu -q > gpurun_out/ab_rslices_pytest.log 2>&1; echo pytest=$?
for i in 1 2 3; do
  timeout 300 python bench.py --only c5g --no-cpu-baseline > gpurun_out/ab_c5g_new$i.json 2>/dev/null
  BS_LIB_PATH=$V timeout 300 python bench.py --only c5g --no-cpu-baseline > gpurun_out/ab_c5g_old$i.json 2>/dev/null
done
python - <<'PY'
import json, statistics
def ld(f): return json.loads([l for l in open(f) if l.startswith("{")][0])
for tag in ("new", "old"):
    g = [ld(f"gpurun_out/ab_c5g_{tag}{i}.json")["c5_greedy"] for i in (1, 2, 3)]
    print(tag, "c5g", ["%.3e" % x["value"] for x in g], "median %.3e" % statistics.median(x["value"] for x in g),
          "d2h", g[0].get("e2e", {}).get("d2h_bytes_per_step"))
PY
