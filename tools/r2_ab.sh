# A/B of library variants: VARIANTS="cur absx/x.so ..." CFGS="c4m c4t"
cp paper_2102_05221_b200/libelastik_b200.so /tmp/cur.so
for v in ${VARIANTS:-cur}; do
  if [ "$v" = cur ]; then cp /tmp/cur.so paper_2102_05221_b200/libelastik_b200.so; else cp $v paper_2102_05221_b200/libelastik_b200.so; fi
  for cfg in ${CFGS:-c2}; do
    timeout 300 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$cfg', round(d['ms_per_step'],3), {a: round(b, 3) for a, b in d['phases_ms'].items() if b > 0.01}, round(d['roofline']['frac'],3))"
  done
done
cp /tmp/cur.so paper_2102_05221_b200/libelastik_b200.so
