#!/bin/bash
# quick GPU check: parity tests + all-config bench summary (run under gpurun)
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 --all --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.log").read().strip().splitlines()[-1])
print("c2", round(d["value"]), round(d["ms_per_step"], 3), {a: round(b, 3) for a, b in d["phases_ms"].items()},
      round(d["roofline"]["frac"], 3), "e2e", round(d.get("e2e", {}).get("value", 0)))
for k, v in d.get("per_config", {}).items():
    print(k, round(v["value"], 2), v["unit"], round(v["ms_per_step"], 3), {a: round(b, 3) for a, b in v["phases_ms"].items()},
          round(v["roofline"]["frac"], 3), v["roofline"]["bound"], v.get("nn_index_mismatch_rate", ""))
PY
