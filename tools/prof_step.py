"""Run one workload's device step a few times (for ncu / compute-sanitizer captures).

    python tools/prof_step.py c2 [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(s)
r = bench.Runner(name, 0, dev)
for _ in range(reps):
    r.step(s.cuda_stream)
torch.cuda.synchronize()
print("ok", name, r.cells_after_step())
