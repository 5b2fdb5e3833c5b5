for mb in 5 6 8; do
  BS_NVCC_EXTRA="-DBS_PREFILL_MINB=$mb -DBS_DECODE_MINB=$mb" python -m paper_2602_18755_b200._build -f > /dev/null
  echo "minb=$mb $(python bench.py --only c4 --no-cpu-baseline | python -c 'import json,sys; d=json.loads(sys.stdin.read())["c4_replay"]; print(d["value"], d["phase_ms_rank0"])')"
done
python -m paper_2602_18755_b200._build -f > /dev/null
python -m pytest tests/test_gpu_cluster_replay.py -x -q 2>&1 | tail -2
