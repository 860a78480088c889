"""Host enqueue cost and device time of one resident step, profiling marks off and on.

    python tools/host_cost.py c2 [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(s)
r = bench.Runner(name, 0, dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(5):
    r.step(s.cuda_stream)
torch.cuda.synchronize()
for prof in (0, 1):
    r.L.ek_set_profiling(prof)
    host, devms = [], []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        t0 = time.perf_counter()
        r.step(s.cuda_stream)
        host.append((time.perf_counter() - t0) * 1e6)
        e1.record(s)
        e1.synchronize()
        devms.append(e0.elapsed_time(e1))
    print(f"{name} profiling={prof}: host enqueue {np.median(host):.1f} us (min {min(host):.1f}), "
          f"device step {np.median(devms):.4f} ms (min {min(devms):.4f})")
    if prof:
        print("  phases", {k: round(v, 4) for k, v in bench.phase_times(r.L).items()})
