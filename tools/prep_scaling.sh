for D in 128 256 512 1024 2048; do
  timeout 300 python bench.py --no-extras --no-cpu-baseline --decisions $D --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($D, {k: round(v,4) for k,v in d['phase_ms_avg'].items()})"
done
