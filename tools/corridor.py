"""Live-corridor widths of the diagonal engine (debug build with -DEKB_LIVE): at every
liveness vote of a C2 phase-B pair, the span of lanes (4 diagonals each) holding a cell
<= the cutoff, per 64 anti-diagonals of t.

    python tools/corridor.py c2      (with the EKB_LIVE library in place)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
dev = torch.device("cuda", 0)
s = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(s)
r = bench.Runner(name, 0, dev)
fn = r.L.ek_debug_corr_dtw
fn.argtypes = [C.POINTER(C.c_ulonglong)]
buf = (C.c_ulonglong * (16 * 33))()
r.step(s.cuda_stream)
torch.cuda.synchronize()
fn(buf)
r.step(s.cuda_stream)
torch.cuda.synchronize()
fn(buf)
h = [[int(buf[b * 33 + k]) for k in range(33)] for b in range(16)]
tot = [sum(h[b][k] for b in range(16)) for k in range(33)]
n = sum(tot)
print(json.dumps({"by_t64": h, "total": tot}))
cum = 0
for k in range(33):
    cum += tot[k]
    print(f"span<={k:2d} lanes: {cum / n:.3f}")

# narrow-window simulation of the same step (EKB_NN2=0 runs the one-pair engine that carries it)
if hasattr(r.L, "ek_debug_sn_dtw"):
    sn = r.L.ek_debug_sn_dtw
    sn.argtypes = [C.POINTER(C.c_ulonglong)]
    b8 = (C.c_ulonglong * 8)()
    sn(b8)
    r.step(s.cuda_stream)
    torch.cuda.synchronize()
    sn(b8)
    names = ["pairs", "narrowed", "overflowed", "votes", "narrow_votes", "narrow_votes_overflowed", "recentrings", "expansions"]
    d = {n: int(b8[k]) for k, n in enumerate(names)}
    d["narrow_share"] = d["narrow_votes"] / max(1, d["votes"])
    print(json.dumps({"narrow_sim": d}))
