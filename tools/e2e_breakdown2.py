"""Where the end-to-end C2 call spends its time (run on the GPU box)."""
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


def med(f, n=10):
    for _ in range(3):
        f()
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t)
    return 1e3 * float(np.median(ts))


# 1. H2D of the same bytes (pinned -> device), torch
dq = torch.empty(Q.shape, dtype=torch.float64, device="cuda")
dc = torch.empty(C.shape, dtype=torch.float64, device="cuda")
tq, tc = torch.from_numpy(Qp), torch.from_numpy(Cp)


def h2d():
    dq.copy_(tq, non_blocking=True)
    dc.copy_(tc, non_blocking=True)
    torch.cuda.synchronize()


print("H2D 17.8 MB ms", round(med(h2d), 3))
# 2. public API
print("nn_batch ms", round(med(lambda: ekb.nn_batch(spec, "eapruned", Qp, Cp)), 3))
# 3. the C call alone with prepared arguments
qf, qo, qlen = Qp.reshape(-1), np.arange(256, dtype=np.int64) * 512, np.full(256, 512, dtype=np.int64)
cf, co, clen = Cp.reshape(-1), np.arange(4096, dtype=np.int64) * 512, np.full(4096, 512, dtype=np.int64)
out = [np.empty(256, dtype=np.int64) for _ in range(5)]
h = _lib.SpecHandle(spec, longest_lengths=[512])


def raw():
    _lib.check(L.ek_nn(h.ref, 2, _lib.dptr(qf), len(qf), _lib.iptr(qo), _lib.iptr(qlen), 256, _lib.dptr(cf), len(cf),
                       _lib.iptr(co), _lib.iptr(clen), 4096, _lib.iptr(out[0]), _lib.dptr(out[1].view(np.float64)),
                       _lib.iptr(out[2]), _lib.iptr(out[3]), _lib.iptr(out[4])))


print("ek_nn ms", round(med(raw), 3))
# 4. device step (inputs resident)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
r = bench.Runner("c2", 0, torch.device("cuda", 0))


def dev():
    r.step(s.cuda_stream)
    torch.cuda.synchronize()


print("device step (host-timed) ms", round(med(dev), 3))
L.ek_set_profiling(1)
raw()
L.ek_set_profiling(0)
print("phases of ek_nn", {k: round(v, 3) for k, v in bench.phase_times(L).items()})
