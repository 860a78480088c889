timeout 900 python bench.py --steps 10 --warmup 3 --all --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.log").read().strip().splitlines()[-1])
print("c2", round(d["value"]), round(d["ms_per_step"], 3), {a: round(b, 3) for a, b in d["phases_ms"].items()}, round(d["roofline"]["frac"], 3))
for k, v in d.get("per_config", {}).items():
    print(k, round(v["value"], 2), round(v["ms_per_step"], 3), {a: round(b, 3) for a, b in v["phases_ms"].items() if b > 0.02}, round(v["roofline"]["frac"], 3), v.get("nn_index_mismatch_rate", ""))
PY
