# Longest C3 probe (bs_simulate_instance) and the C3 table: default library vs a variant, alternating.
V=$PWD/paper_2602_18755_b200/libbiscale_gpu_$1.so
for i in 1 2; do
  python tools/decode_probe_profile.py 2>&1 | tail -1 | sed 's/^/base /'
  BS_LIB_PATH=$V python tools/decode_probe_profile.py 2>&1 | tail -1 | sed "s/^/$1 /"
done
