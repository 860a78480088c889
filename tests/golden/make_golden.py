"""Generate golden fixtures from the LIVE reference package (run in the build container).

    python tests/golden/make_golden.py

Imports /root/reference/pkg/src/elastik with its own compiled kernel
(oracle/_ref, built by `make -C oracle ref`) and records, with fixed seeds:

  pairs.npz     -- engines.distance for every kind x cost mode x variant over
                   random pairs of random lengths / windows / parameters and
                   cutoffs {inf, 1.05, 1.0, 0.95, 0.3} x exact (the sweep of
                   pkg/tests/test_backends.py:30-55), costs and cell counts;
  nn.npz        -- classify_1nn on small warped-prototype datasets per kind;
  pairwise.npz  -- the pruned_only all-pairs matrix for wdtw and erp;
  subseq.npz    -- subsequence_search (raw and z-normalised) for dtw / cdtw.

The fixtures travel to the GPU box; /root/reference does not.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)

import refpkg  # noqa: E402

ek = refpkg.load()
assert ek is not None, "reference package not found"
assert ek.compiled_available(), "build oracle/_ref first: make -C oracle ref"

from paper_2102_05221_b200 import datagen  # noqa: E402

KINDS = ek.KINDS
VARIANTS = ("base", "ea", "eapruned", "pruned_only")


def spec_dict(spec):
    return {k: getattr(spec, k) for k in ("kind", "window", "wdtw_g", "erp_gap", "msm_c", "twe_nu", "twe_lambda",
                                          "cost_mode")}


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


def make_pairs(seed=20241020, per=14):
    rng = np.random.default_rng(seed)
    series, specs, rows = [], [], []
    for kind in KINDS:
        for mode in ("squared", "absolute"):
            for _ in range(per):
                la, lb = int(rng.integers(1, 48)), int(rng.integers(1, 48))
                spec = random_spec(kind, rng, max(la, lb), mode)
                if rng.random() < 0.5:
                    a = np.cumsum(rng.normal(0, 1, la))
                    b = np.cumsum(rng.normal(0, 1, lb))
                else:
                    a = rng.uniform(-4, 4, la)
                    b = rng.uniform(-4, 4, lb)
                ia = len(series); series.append(a)
                ib = len(series); series.append(b)
                si = len(specs); specs.append(spec_dict(spec))
                exact = ek.distance(spec, "base", a, b).cost
                cutoffs = [math.inf]
                if math.isfinite(exact) and exact > 0:
                    cutoffs += [exact * f for f in (1.05, 1.0, 0.95, 0.3)]
                for v in VARIANTS:
                    for co in cutoffs:
                        r = ek.distance(spec, v, a, b, cutoff=co)
                        rows.append((si, ia, ib, VARIANTS.index(v), co, r.cost, r.cells_computed))
    lens = np.array([len(s) for s in series], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    r = np.array(rows, dtype=object)
    return dict(series=np.concatenate(series), series_off=off, series_len=lens,
                specs=json.dumps(specs), spec_idx=r[:, 0].astype(np.int64), a=r[:, 1].astype(np.int64),
                b=r[:, 2].astype(np.int64), variant=r[:, 3].astype(np.int64), cutoff=r[:, 4].astype(np.float64),
                cost=r[:, 5].astype(np.float64), cells=r[:, 6].astype(np.int64))


NN_SPECS = [
    ek.DistanceSpec(kind="dtw"),
    ek.DistanceSpec(kind="cdtw", window=6),
    ek.DistanceSpec(kind="wdtw", wdtw_g=0.05),
    ek.DistanceSpec(kind="erp", window=5, erp_gap=0.0),
    ek.DistanceSpec(kind="msm", msm_c=1.0),
    ek.DistanceSpec(kind="twe", twe_nu=0.001, twe_lambda=1.0),
    ek.DistanceSpec(kind="cdtw", window=4, cost_mode="absolute"),
]


def make_nn():
    out = {"specs": json.dumps([spec_dict(s) for s in NN_SPECS])}
    for k, spec in enumerate(NN_SPECS):
        X, y, _ = datagen.warped_prototypes(40, 48, 4, 0.2, 777 + k)
        Q, qy, _ = datagen.warped_prototypes(12, 48, 4, 0.2, 888 + k)
        train = ek.LabeledDataset("train", tuple((int(a), b) for a, b in zip(y, X)))
        test = ek.LabeledDataset("test", tuple((int(a), b) for a, b in zip(qy, Q)))
        recs = ek.classify_1nn(train, test, ek.SearchConfig(spec=spec, variant="eapruned"))
        out[f"X{k}"], out[f"y{k}"], out[f"Q{k}"], out[f"qy{k}"] = X, y, Q, qy
        out[f"idx{k}"] = np.array([r.nn_index for r in recs], dtype=np.int64)
        out[f"dist{k}"] = np.array([r.nn_distance for r in recs])
        out[f"pred{k}"] = np.array([r.predicted for r in recs], dtype=np.int64)
    # ties: duplicated candidates must resolve to the lowest index
    X, y, _ = datagen.warped_prototypes(10, 32, 2, 0.1, 999)
    Xd = np.concatenate([X, X[::-1]])
    spec = ek.DistanceSpec(kind="dtw")
    recs = ek.classify_1nn(ek.LabeledDataset("t", tuple((0, s) for s in Xd)),
                           ek.LabeledDataset("q", tuple((0, s) for s in X)), ek.SearchConfig(spec=spec))
    out["tie_X"], out["tie_Q"] = Xd, X
    out["tie_idx"] = np.array([r.nn_index for r in recs], dtype=np.int64)
    out["tie_dist"] = np.array([r.nn_distance for r in recs])
    return out


def make_pairwise():
    out = {}
    X, _, _ = datagen.warped_prototypes(24, 40, 3, 0.1, 4242)
    for name, spec in (("wdtw", ek.DistanceSpec(kind="wdtw", wdtw_g=0.05)),
                       ("erp", ek.DistanceSpec(kind="erp", window=4, erp_gap=0.0))):
        n = len(X)
        D = np.zeros((n, n))
        for i in range(n):
            for j in range(i + 1, n):
                D[i, j] = D[j, i] = ek.distance(spec, "pruned_only", X[i], X[j]).cost
        out[f"D_{name}"] = D
    out["X"] = X
    return out


def make_subseq():
    rng = np.random.default_rng(1234)
    ref = np.cumsum(rng.normal(0, 1, 600))
    q = np.cumsum(rng.normal(0, 1, 40))
    out = {"ref": ref, "q": q}
    cases = [("dtw", None, False), ("dtw", None, True), ("cdtw", 3, True), ("cdtw", 8, False)]
    res = []
    for kind, w, norm in cases:
        spec = ek.DistanceSpec(kind=kind, window=w)
        off, d, _ = ek.subsequence_search(q, ref, ek.SearchConfig(spec=spec, variant="eapruned", normalize=norm))
        res.append((off, d))
    out["cases"] = json.dumps([list(c) for c in cases])
    out["off"] = np.array([r[0] for r in res], dtype=np.int64)
    out["dist"] = np.array([r[1] for r in res])
    return out


def main():
    np.savez_compressed(os.path.join(HERE, "pairs.npz"), **make_pairs())
    np.savez_compressed(os.path.join(HERE, "nn.npz"), **make_nn())
    np.savez_compressed(os.path.join(HERE, "pairwise.npz"), **make_pairwise())
    np.savez_compressed(os.path.join(HERE, "subseq.npz"), **make_subseq())
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
