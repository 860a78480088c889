python tools/host_cost.py c2 30 2>&1 | tail -3
python bench.py --no-cpu-baseline > gpurun_out/s5_c.json 2>/dev/null; python - <<'PY'
import json
d=json.loads(open("gpurun_out/s5_c.json").read().strip().splitlines()[-1])
print(d["value"],d["ms_per_step"],d["phases_ms"],d["roofline"]["frac"],d["e2e"]["value"],d["e2e_sync"]["value"],d["gpu_launches"])
PY
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
