"""Live share of the cells the diagonal engine evaluates (debug build with -DEKB_LIVE):
evaluated in-matrix band cells vs those whose value was <= the cutoff in force -- the cells
EAPruned's per-row pruning (_speedups.pyx:184-263) would still compute.

    python tools/live_cells.py c2 c4m c4t      (with the EKB_LIVE library in place)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

out = {}
for name in sys.argv[1:] or ["c2"]:
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(s)
    r = bench.Runner(name, 0, dev)
    kind = {"c2": "dtw", "c1": "dtw", "c4m": "msm", "c4t": "twe"}[name]
    fn = getattr(r.L, f"ek_debug_live_{kind}")
    fn.argtypes = [C.POINTER(C.c_ulonglong)]
    buf = (C.c_ulonglong * 2)()
    r.step(s.cuda_stream)
    torch.cuda.synchronize()
    fn(buf)  # reset
    r.step(s.cuda_stream)
    torch.cuda.synchronize()
    fn(buf)
    ev, live = int(buf[0]), int(buf[1])
    out[name] = {"evaluated_band_cells": ev, "live_cells": live, "live_fraction": live / max(1, ev),
                 "engine_cells_reported": r.cells_after_step()}
    print(name, out[name], flush=True)
print(json.dumps(out))
