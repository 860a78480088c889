"""Per-phase device times of one end-to-end nn_batch call (C2), host arrays pinned."""
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
L = _lib.lib()
for _ in range(3):
    ekb.nn_batch(spec, "eapruned", Qp, Cp)
ts = []
for _ in range(10):
    t = time.perf_counter()
    ekb.nn_batch(spec, "eapruned", Qp, Cp)
    ts.append(time.perf_counter() - t)
L.ek_set_profiling(1)
ekb.nn_batch(spec, "eapruned", Qp, Cp)
L.ek_set_profiling(0)
print("chunks", os.environ.get("EKB_NN_CHUNKS", "default"), "nn_batch ms", round(1e3 * np.median(ts), 3),
      {k: round(v, 3) for k, v in bench.phase_times(L).items()})
