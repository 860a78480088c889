# A/B of prebuilt library variants in abso/ (run under gpurun)
cp paper_2102_05221_b200/libelastik_b200.so /tmp/cur.so
for v in ${VARIANTS:-old new}; do
  cp abso/$v.so paper_2102_05221_b200/libelastik_b200.so
  for cfg in ${CFGS:-c2 c4t}; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$cfg', round(d['ms_per_step'],3), {a: round(b, 3) for a, b in d['phases_ms'].items()})"
  done
done
cp /tmp/cur.so paper_2102_05221_b200/libelastik_b200.so
