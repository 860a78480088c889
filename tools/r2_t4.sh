D=gpurun_out/t4; mkdir -p $D
run() { timeout 300 env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step'],4), round(d['phases_ms']['nn_phaseB'],4), round(d['roofline']['frac'],3))"; }
run EKB_NN_SEG1=64
run EKB_NN_SEG1=128
run EKB_NN_SEG1=256
run EKB_NN_SEG1=128 EKB_NN_K2=8
run EKB_NN_SEG1=256 EKB_NN_K2=16
run EKB_NN_SEG1=384 EKB_NN_K2=8
run EKB_NN_SEG1=4096
