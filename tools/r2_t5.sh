run() { timeout 300 env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step'],4), round(d['phases_ms']['nn_phaseB'],4))"; }
run EKB_NN_XSMEM=0
run EKB_NN_XSMEM=12000
run EKB_NN_XSMEM=30000
run EKB_NN_XSMEM=60000
