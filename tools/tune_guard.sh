# guarded-band width sweep on the C4 configs (run under gpurun)
for g in 8 16; do for c in c4m c4t; do EKB_GUARD=$g timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g_${g}_$c.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/g_${g}_$c.log').read().strip().splitlines()[-1]);print('$g', '$c', round(d['ms_per_step'],2), {a: round(v,2) for a,v in d['phases_ms'].items()})"; done; done
