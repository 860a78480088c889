"""Per-warp timeline of k_nn2 (debug build with -DEKB_TRACE): end-time spread, busy share of
the half-warp pair slots, blocks and pairs per warp.

    python tools/trace_nn2.py c2
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(s)
r = bench.Runner(name, 0, dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(3):
    flush.zero_()
    r.step(s.cuda_stream)
torch.cuda.synchronize()
L = r.L
L.ek_debug_trace.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * (8192 * 8))()
L.ek_debug_trace(buf, 8192 * 8)
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8).astype(np.float64)
a = a[a[:, 1] > 0]
t0 = a[:, 0].min()
st, en, busy, blocks, pairs = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2], a[:, 3], a[:, 4]
print(f"{name}: warps {len(a)}  launch span {en.max():.1f} us  start spread {st.max():.1f} us")
print("end pct (us):", np.percentile(en, [0, 10, 25, 50, 75, 90, 99, 100]).round(1))
print("busy share of half slots over blocks:", round(float(busy.sum() / (2 * blocks.sum())), 3))
print("blocks per warp pct:", np.percentile(blocks, [0, 10, 50, 90, 100]), " pairs per warp pct:",
      np.percentile(pairs, [0, 10, 50, 90, 100]), " total pairs", pairs.sum())
act = np.zeros(int(en.max()) + 2)
for x, y in zip(st, en):
    act[int(x):int(y) + 1] += 1
print("active warps over time (every 10%):", [int(act[int(f * en.max())]) for f in np.linspace(0, 0.99, 11)])
exh, lastp = (a[:, 5] - t0) / 1e3, (a[:, 6] - t0) / 1e3
print("work exhausted at pct (us):", np.percentile(exh, [0, 10, 50, 90, 100]).round(1))
print("last pair started pct (us):", np.percentile(lastp, [0, 10, 50, 90, 100]).round(1))
print("drain (end - last pair start) pct (us):", np.percentile(en - lastp, [0, 10, 50, 90, 99, 100]).round(1))
