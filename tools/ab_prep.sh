# headline (prepare phase) and the controller call: default library vs a variant; MPC parity tests
bash tools/ab_variant.sh $1
for v in base $1 base $1; do
  L=""; [ "$v" != base ] && L=$PWD/paper_2602_18755_b200/libbiscale_gpu_$v.so
  env ${L:+BS_LIB_PATH=$L} python tools/c1_latency.py | sed "s/^/$v /"
done
timeout 900 python -m pytest -q -m gpu tests/test_gpu_mpc.py tests/test_golden.py -x 2>&1 | tail -1
