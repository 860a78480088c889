"""Where the end-to-end nn_batch time goes (host side), for the C2 workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2102_05221_b200 as ekb  # noqa: E402
from paper_2102_05221_b200 import _lib, search  # noqa: E402

wl, Q, ql, C, cl = bench.nn_data("c2")
Qp, Cp = bench.pinned_copy(Q), bench.pinned_copy(C)
spec = ekb.DistanceSpec(kind="cdtw", window=51)
for _ in range(3):
    ekb.nn_batch(spec, "eapruned", Qp, Cp)
T = {}
def tick(name, t0):
    T[name] = T.get(name, 0.0) + time.perf_counter() - t0
for _ in range(10):
    t = time.perf_counter(); qf = search._pack(Qp); cf = search._pack(Cp); tick("pack+isfinite", t)
    t = time.perf_counter(); h = _lib.SpecHandle(spec, longest_lengths=[512]); tick("spec", t)
    t = time.perf_counter(); ekb.nn_batch(spec, "eapruned", Qp, Cp); tick("nn_batch total", t)
    t = time.perf_counter(); np.isfinite(Cp).all(); tick("isfinite C", t)
print({k: round(v / 10 * 1e3, 3) for k, v in T.items()}, "ms")
