# quick: device step of the given configs, no CPU baseline / e2e
for cfg in ${CFGS:-c2}; do
timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],4), {a: round(b, 3) for a, b in d['phases_ms'].items() if b > 0.005}, round(d['roofline']['frac'],3))"
done
