# A/B of the C2 step: k_nn2 (default) vs the one-pair-per-warp k_nn (EKB_NN2=0)
for v in 1 0 1; do
  EKB_NN2=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('NN2=$v', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['phases_ms'].items()}, d.get('parity'))"
done
