"""Streaming 1-NN (NNPipeline) on the C2 workload: wall time per step for several stream
lengths, the synchronous call, and the device time of one search without an L2 flush."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2102_05221_b200 as ekb  # noqa: E402
from paper_2102_05221_b200 import _lib  # noqa: E402

wl, Q, ql, C, cl = bench.nn_data("c2")
Qp, Cp = bench.pinned_copy(Q), bench.pinned_copy(C)
spec = ekb.DistanceSpec(kind="cdtw", window=51)
for _ in range(3):
    ekb.nn_batch(spec, "eapruned", Qp, Cp)
    list(ekb.nn_batch_stream(spec, "eapruned", [(Qp, Cp)] * 3))
t = []
for _ in range(10):
    t0 = time.perf_counter()
    ekb.nn_batch(spec, "eapruned", Qp, Cp)
    t.append(time.perf_counter() - t0)
print(f"sync call: {np.mean(t) * 1e3:.3f} ms")
for k in (2, 5, 10, 30, 100):
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in ekb.nn_batch_stream(spec, "eapruned", ((Qp, Cp) for _ in range(k))):
            pass
        ts.append((time.perf_counter() - t0) / k)
    print(f"stream k={k}: {np.mean(ts) * 1e3:.3f} ms/step  ({256 / np.mean(ts):.0f} q/s)")
# host cost of submit and collect alone
pipe = ekb.NNPipeline(spec, "eapruned")
ts, tc = [], []
for _ in range(10):
    t0 = time.perf_counter(); pipe.submit(Qp, Cp); ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize(); time.sleep(0.003)
    t0 = time.perf_counter(); pipe.collect(); tc.append(time.perf_counter() - t0)
print(f"host submit {np.mean(ts) * 1e6:.0f} us, collect after completion {np.mean(tc) * 1e6:.0f} us")
# the device search alone, back to back on resident inputs (no L2 flush, no copies)
r = bench.Runner("c2", 0, torch.device("cuda:0"))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        r.step(s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        r.step(s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
print(f"device back-to-back (no flush): {e0.elapsed_time(e1) / 20:.3f} ms/step")
