# Exhaustive MPC parity tests, then C2 / loose C2 / C5x: default library vs a variant (tools/ab_exh.sh VARIANT)
timeout 900 python -m pytest tests/test_gpu_mpc.py tests/test_golden.py tests/test_gpu_exhaustive_deep.py -x -q > gpurun_out/pytest_x.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_x.log
bash tools/ab_variant.sh $1
bash tools/ab_variant.sh $1 --ttft 1200
for v in base $1; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} timeout 600 python bench.py --only c5x --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c5x', round(d['c5_exhaustive']['value']))"
done
