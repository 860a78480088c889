"""Record the native-seam calls of the LIVE reference (run in the build container):

    python tests/golden/make_golden_dispatch.py

The reference's only native seam is ``_speedups.run`` (pkg/src/elastik/_speedups.pyx:274-317),
called by ``engines._dispatch`` (pkg/src/elastik/engines.py:29-50).  This script wraps the
reference's compiled ``run`` (oracle/_ref, built from its .pyx) with a recorder and drives the
reference's own public API:

* ``engines.distance`` for every kind x cost mode x variant (base / ea / eapruned /
  pruned_only), equal and unequal lengths, cutoffs {inf, 1.05, 1, 0.95, 0.3} x exact --
  so compute_base's ``window=0`` calls, the windowed base, the diagonal-bound cutoffs of
  pruned_only and infeasible windows all appear as the reference issues them;
* ``compute_ea`` / ``compute_eapruned`` on ``make_recurrence(orient="st")`` pairs with the
  shorter series on the rows;
* ``nn_search`` on a small set (running-best cutoffs).

dispatch.npz holds every call's arguments (engine, lines, cols, kind, mode, window, cutoff,
erp_gap, msm_c, twe_nu, twe_lambda, weights, vborder_vals, hborder_vals) and its return value
(cost, cells).  tests/test_gpu_seam.py replays them through paper_2102_05221_b200.speedups.run.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import refpkg  # noqa: E402

ek = refpkg.load()
assert ek is not None, "reference package not found"
assert ek.compiled_available(), "build oracle/_ref first: make -C oracle ref"

from elastik import _backend, engines  # noqa: E402
from elastik.kernels import make_recurrence  # noqa: E402

_real = _backend.speedups()
CALLS = []


class _Recorder:
    EMPTY = _real.EMPTY

    @staticmethod
    def run(engine, lines, cols, kind, mode, window, cutoff, gap, c, nu, lam, weights, vb, hb):
        out = _real.run(engine, lines, cols, kind, mode, window, cutoff, gap, c, nu, lam, weights, vb, hb)
        CALLS.append((engine, np.array(lines), np.array(cols), kind, mode, window, cutoff, gap, c, nu, lam,
                      np.array(weights), np.array(vb), np.array(hb), out[0], out[1]))
        return out


_backend._speedups = _Recorder  # _dispatch reads it through _backend.speedups()


def random_spec(kind, rng, maxlen, mode):
    if kind == "dtw":
        return ek.DistanceSpec(kind="dtw", cost_mode=mode)
    if kind == "cdtw":
        return ek.DistanceSpec(kind="cdtw", window=int(rng.integers(0, maxlen + 1)), cost_mode=mode)
    if kind == "wdtw":
        return ek.DistanceSpec(kind="wdtw", wdtw_g=float(rng.uniform(0.0, 0.6)), cost_mode=mode)
    if kind == "erp":
        return ek.DistanceSpec(kind="erp", window=int(rng.integers(0, maxlen + 1)),
                               erp_gap=float(rng.uniform(-1.0, 1.0)), cost_mode=mode)
    if kind == "msm":
        return ek.DistanceSpec(kind="msm", msm_c=float(rng.uniform(0.0, 2.0)), cost_mode=mode)
    return ek.DistanceSpec(kind="twe", twe_nu=float(rng.uniform(0.0, 1.0)),
                           twe_lambda=float(rng.uniform(0.0, 2.0)), cost_mode=mode)


def main():
    rng = np.random.default_rng(8675309)
    for kind in ek.KINDS:
        for mode in ("squared", "absolute"):
            for k in range(6):
                la = int(rng.integers(1, 40))
                lb = la if k < 2 else int(rng.integers(1, 40))  # equal and unequal lengths
                spec = random_spec(kind, rng, max(la, lb), mode)
                a = np.cumsum(rng.normal(0, 1, la))
                b = np.cumsum(rng.normal(0, 1, lb))
                exact = ek.distance(spec, "base", a, b).cost
                cuts = [math.inf] + ([exact * f for f in (1.05, 1.0, 0.95, 0.3)] if 0 < exact < math.inf else [])
                for v in ("base", "ea", "eapruned", "pruned_only"):
                    for co in cuts:
                        ek.distance(spec, v, a, b, cutoff=co)
                # orient="st": the shorter series on the rows, through compute_ea / compute_eapruned
                s, t = (a, b) if la <= lb else (b, a)
                rec = make_recurrence(spec, s, t, orient="st")
                w = int(rng.integers(0, max(len(s), len(t)) + 1))
                engines.compute_base(rec)
                for co in (math.inf, 3.0, 30.0):
                    engines.compute_ea(rec, w, co)
                    engines.compute_eapruned(rec, w, co)
    # nn_search: the running best as the cutoff
    X = [np.cumsum(rng.normal(0, 1, 24)) for _ in range(30)]
    q = np.cumsum(rng.normal(0, 1, 24))
    for spec in (ek.DistanceSpec(kind="cdtw", window=3), ek.DistanceSpec(kind="msm", msm_c=0.5)):
        ek.nn_search(q, X, ek.SearchConfig(spec=spec, variant="eapruned"))
        ek.nn_search(q, X, ek.SearchConfig(spec=spec, variant="ea"))
    arr = lambda k: [c[k] for c in CALLS]  # noqa: E731
    cat = lambda k: np.concatenate(arr(k)) if any(len(x) for x in arr(k)) else np.zeros(0)  # noqa: E731
    lens = lambda k: np.array([len(x) for x in arr(k)], dtype=np.int64)  # noqa: E731
    np.savez_compressed(
        os.path.join(HERE, "dispatch.npz"),
        engine=np.array(arr(0)), lines=cat(1), lines_len=lens(1), cols=cat(2), cols_len=lens(2),
        kind=np.array(arr(3), dtype=np.int64), mode=np.array(arr(4), dtype=np.int64),
        window=np.array(arr(5), dtype=np.int64), cutoff=np.array(arr(6), dtype=np.float64),
        params=np.array([c[7:11] for c in CALLS], dtype=np.float64),
        weights=cat(11), weights_len=lens(11), vb=cat(12), vb_len=lens(12), hb=cat(13), hb_len=lens(13),
        cost=np.array(arr(14), dtype=np.float64), cells=np.array(arr(15), dtype=np.int64))
    engs = arr(0)
    print(f"recorded {len(CALLS)} _speedups.run calls "
          f"({engs.count('base')} base, {engs.count('ea')} ea, {engs.count('eapruned')} eapruned; "
          f"{sum(len(c[1]) < len(c[2]) for c in CALLS)} with shorter rows)")


if __name__ == "__main__":
    main()
