BS_LIB_PATH=$PWD/paper_2602_18755_b200/libbiscale_gpu_pph.so timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/pph.json 2> gpurun_out/pph.err
BS_LIB_PATH=$PWD/paper_2602_18755_b200/libbiscale_gpu_pph.so timeout 300 python tools/c2_e2e_timing.py > gpurun_out/pph2.log 2>&1
