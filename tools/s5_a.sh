set -x
python tools/host_cost.py c2 30 2>&1 | tail -4
EKB_WORKSPACE=0 python tools/host_cost.py c2 30 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
