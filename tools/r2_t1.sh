set -x
D=gpurun_out/t1; mkdir -p $D
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/c2.json 2> $D/c2.err
timeout 200 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $D/c1.json 2> $D/c1.err
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/pytest.log 2>&1
tail -5 $D/pytest.log
python -c "
import json
for n in ('c2','c1'):
    d=json.loads(open('$D/'+n+'.json').read().strip().splitlines()[-1]); print(n, round(d['value']), round(d['ms_per_step'],4), {a:round(b,3) for a,b in d['phases_ms'].items()}, round(d['roofline']['frac'],3))
"
