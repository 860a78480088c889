timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in c4m; do python tools/host_cost.py $cfg 3 2>&1 | tail -2; done
