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

# the long pairs (>= 400 anti-diagonals) of the last launches: when they started, how long
# they ran, their query and key / threshold ratio at the start
if hasattr(L, "ek_debug_plog"):
    L.ek_debug_plog.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    L.ek_debug_plog(None, 0)  # reset
    flush.zero_()
    r.step(s.cuda_stream)
    torch.cuda.synchronize()
    pb = (C.c_ulonglong * (32768 * 4))()
    n = L.ek_debug_plog(pb, 32768)
    L.ek_debug_trace(buf, 8192 * 8)
    a2 = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8).astype(np.float64)
    a2 = a2[a2[:, 1] > 0]
    t0 = a2[:, 0].min()
    span = (a2[:, 1].max() - t0) / 1e3
    p = np.frombuffer(pb, dtype=np.uint64).reshape(-1, 4)[:n]
    ps, pe = (p[:, 0].astype(np.float64) - t0) / 1e3, (p[:, 1].astype(np.float64) - t0) / 1e3
    q, te = (p[:, 2] >> np.uint64(32)).astype(np.int64), (p[:, 2] & np.uint64(0xffffffff)).astype(np.int64)
    ratio = p[:, 3].astype(np.float64) / 1e6
    print(f"long pairs (tend >= 400): {n}  launch span {span:.1f} us")
    for lo, hi in ((0, 100), (100, 200), (200, 300), (300, 350), (350, 400), (400, 450), (450, 1e9)):
        m = (ps >= lo) & (ps < hi)
        if m.sum():
            print(f"  started in [{lo}, {hi}) us: {int(m.sum())} pairs, full-length {int((te[m] >= 1024).sum())}, "
                  f"duration median {np.median(pe[m] - ps[m]):.1f} max {np.max(pe[m] - ps[m]):.1f} us, "
                  f"key/thr median {np.median(ratio[m]):.3f} (10% {np.percentile(ratio[m], 10):.3f}, "
                  f"90% {np.percentile(ratio[m], 90):.3f}), distinct queries {len(np.unique(q[m]))}")
    late = ps >= 350
    if late.sum():
        uq, cnt = np.unique(q[late], return_counts=True)
        o = np.argsort(-cnt)[:12]
        print("  queries of the late long pairs (query: count):", {int(uq[k]): int(cnt[k]) for k in o})
        print("  end times of late long pairs pct:", np.percentile(pe[late], [50, 90, 99, 100]).round(1))
