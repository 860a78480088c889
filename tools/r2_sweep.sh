# env sweep of the LB-path schedule on C2 (run under gpurun)
for e in "EKB_NN_K2=4" "EKB_NN_K2=2" "EKB_NN_K2=8" "EKB_NN_SEG1=32" "EKB_NN_SEG1=128" "EKB_NN_SEEDS=32"; do
  env $e timeout 300 python bench.py --config c2 --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$e', round(d['ms_per_step'],4), {a: round(b, 4) for a, b in d['phases_ms'].items() if b > 0.01})"
done
