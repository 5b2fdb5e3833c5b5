# ncu source profile of the C3 table's longest decode probe (tools/decode_probe_profile.py)
set -x
timeout 300 python tools/decode_probe_profile.py > gpurun_out/dpp_pre.log 2>&1; echo pre=$?
ncu --set full --clock-control none --import-source on -k regex:sim_kernel -s 1 -c 1 -o gpurun_out/dpp_full python tools/decode_probe_profile.py > gpurun_out/dpp_full.log 2>&1; echo ncu=$?
