# A/B of bulk (TMA) candidate staging on the C4 configs (run under gpurun)
for c in c4t c4m; do for b in 1 0; do
  EKB_BULK=$b timeout 600 python bench.py --config $c --steps ${STEPS:-3} --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c bulk=$b', round(d['ms_per_step'],3), {a: round(b, 3) for a, b in d['phases_ms'].items() if b > 0.01}, round(d['roofline']['frac'],3))"
done; done
