CFGS="c2 c3e c4t" bash tools/r2_q.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_seam.py -x -q -p no:cacheprovider 2>&1 | tail -2
