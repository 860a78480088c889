D=gpurun_out/t3; mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullshape.py -x -q -p no:cacheprovider -k "nn or c2 or halves" > $D/pytest.log 2>&1
tail -3 $D/pytest.log
for s in 1 2; do EKB_NN_SPLIT=$s timeout 300 python tools/e2e_phases.py; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $D/c2.json 2> $D/c2.err
python -c "
import json; d=json.loads(open('$D/c2.json').read().strip().splitlines()[-1]); print(round(d['value']), d['e2e'])"
