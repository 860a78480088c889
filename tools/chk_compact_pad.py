"""Equal-length all-pairs on the half-warp diagonal engine (compact pads), every kind, against
the oracle; with a -DEKB_BOUNDS=40 build any staged-series read beyond 40 elements traps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2102_05221_b200 as ekb  # noqa: E402
from oracle import eko  # noqa: E402

rng = np.random.default_rng(5)
specs = [ekb.DistanceSpec(kind="cdtw", window=25), ekb.DistanceSpec(kind="erp", erp_gap=0.0, window=25),
         ekb.DistanceSpec(kind="erp", erp_gap=0.3, window=30), ekb.DistanceSpec(kind="msm", msm_c=0.7, window=12),
         ekb.DistanceSpec(kind="twe", twe_nu=0.01, twe_lambda=0.4, window=29),
         ekb.DistanceSpec(kind="wdtw", wdtw_g=0.05, window=20), ekb.DistanceSpec(kind="cdtw", window=0),
         ekb.DistanceSpec(kind="cdtw", window=29, cost_mode="absolute")]
for L in (2, 3, 17, 64, 255, 256, 300):
    X = np.cumsum(rng.standard_normal((13, L)), axis=1)
    for spec in specs:
        print("L", L, spec.kind, spec.window, flush=True)
        D = ekb.pairwise(spec, X, variant="pruned_only")
        D = D[0] if isinstance(D, tuple) else D
        want = eko.pairwise(spec, X, "pruned_only")
        want = want[0] if isinstance(want, tuple) else want
        if not np.array_equal(D, want):
            print("MISMATCH", L, spec.kind, spec.window, D[0, :4], want[0, :4])
print("compact pads ok")
