# A/B of the block-shared |i-j| table on C3 WDTW (run under gpurun)
for v in 1 0; do
  EKB_SHARED_TAB=$v timeout 600 python bench.py --config c3w --steps ${STEPS:-5} --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3w shared=$v', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d.get('parity'))"
done
