"""GPU: the optional FP32 mode (BASELINE.json north star: "An optional FP32 mode must
stay within 1e-5 relative of the reference, with the NN-index mismatch rate
reported").

The FP32 engines are the FP64 engines instantiated on float (inputs rounded to
float once, the same recurrence, cutoff rounded down so keep-if-<= is exact in
float).  Tolerance, written here: |d32 - d64| <= 1e-5 * d64, d64 from the CPU
oracle (the reference's algorithm).  1-NN answers may differ from the reference
only on near ties; the mismatch rate is printed and bounded, and every mismatch
must be a near tie (the reference's exact distance of the FP32 pick within 2e-5
of the best).
"""

import math

import numpy as np
import pytest

from oracle import eko
from test_gpu_parity import _workload_rows, random_spec

pytestmark = pytest.mark.gpu

RTOL = 1e-5


def rel_ok(got, want, rtol=RTOL):
    if math.isinf(want) or math.isinf(got):
        return math.isinf(want) and math.isinf(got)
    return abs(got - want) <= rtol * abs(want)


def walk(rng, n):
    x = np.cumsum(rng.normal(0, 1, n))
    return (x - x.mean()) / (x.std() + 1e-12)


@pytest.mark.parametrize("kind", ["dtw", "cdtw", "wdtw", "erp", "msm", "twe"])
@pytest.mark.parametrize("mode", ["squared", "absolute"])
def test_fp32_distance_sweep(gpu, kind, mode):
    """Lengths 8..300 (diagonal and row-stripe engines, every band shape): base within
    1e-5; eapruned / pruned_only finite within 1e-5 under cutoff 1.05x, +inf under 0.95x;
    ea finite within 1e-5 under 1.05x (every row minimum <= the cost)."""
    rng = np.random.default_rng(hash(("fp32", kind, mode)) % 2**32)
    bad, worst = [], 0.0
    for trial in range(40):
        hi = 48 if trial < 25 else 300
        la, lb = int(rng.integers(8, hi)), int(rng.integers(8, hi))
        spec = random_spec(gpu, kind, rng, max(la, lb), mode)
        a, b = walk(rng, la), walk(rng, lb)
        exact = eko.distance(spec, "base", a, b)[0]
        got, _ = gpu.distance_batch(spec, "base", [(a, b)], precision="float32")
        if not rel_ok(got[0], exact):
            bad.append(("base", la, lb, spec.window, got[0], exact))
        if math.isfinite(exact) and exact > 0:
            worst = max(worst, abs(got[0] - exact) / exact)
            for v, f, fin in (("eapruned", 1.05, True), ("eapruned", 0.95, False), ("ea", 1.05, True),
                              ("pruned_only", math.inf, True)):
                want = eko.distance(spec, v, a, b, exact * f)[0]
                c, _ = gpu.distance_batch(spec, v, [(a, b)], cutoffs=[exact * f], precision="float32")
                if fin and not rel_ok(c[0], want):
                    bad.append((v, f, la, lb, spec.window, c[0], want))
                if not fin and not math.isinf(c[0]):
                    bad.append((v, f, la, lb, spec.window, c[0], want))
    print(f"fp32 {kind}/{mode}: max relative error {worst:.3g}")
    assert not bad, bad[:8]


@pytest.mark.parametrize("which", ["c2", "c4m", "c4t"])
def test_fp32_nn_benchmark_shapes(gpu, which):
    """BASELINE shapes (full candidate sets) on a query subset: FP32 1-NN distances
    within 1e-5 of the reference's; NN-index mismatches are near ties and rare."""
    from paper_2102_05221_b200 import datagen

    wl = datagen.C2 if which == "c2" else datagen.C4
    nq = 32 if which == "c2" else 8
    Q, C = _workload_rows(wl, nq, seed_shift=7)
    spec = {"c2": gpu.DistanceSpec(kind="cdtw", window=51),
            "c4m": gpu.DistanceSpec(kind="msm", msm_c=1.0),
            "c4t": gpu.DistanceSpec(kind="twe", twe_nu=0.001, twe_lambda=1.0)}[which]
    idx, dist = gpu.nn_batch(spec, "eapruned", Q, C, precision="float32")[:2]
    r = eko.nn(spec, "eapruned", Q, C, threads=16)
    mism = idx != r["nn_index"]
    print(f"fp32 {which}: NN-index mismatch rate {mism.mean():.4f} ({int(mism.sum())}/{nq})")
    bad = []
    for q in range(nq):
        if not rel_ok(dist[q], r["nn_distance"][q]):
            bad.append(("dist", q, dist[q], r["nn_distance"][q]))
        if mism[q]:
            alt = eko.distance(spec, "base", Q[q], C[idx[q]])[0]
            if not rel_ok(alt, r["nn_distance"][q], 2 * RTOL):
                bad.append(("not a near tie", q, int(idx[q]), int(r["nn_index"][q]), alt, r["nn_distance"][q]))
    assert not bad, bad[:6]
    assert mism.mean() <= 0.1


def test_fp32_nn_variants_agree(gpu, rng):
    """base / ea / eapruned / pruned_only give the same FP32 1-NN answer (the shared
    cutoff, LB pre-test and seeds are exact in float), ragged lengths included."""
    spec = gpu.DistanceSpec(kind="cdtw", window=9)
    Q = [walk(rng, int(rng.integers(40, 90))) for _ in range(6)]
    C = [walk(rng, int(rng.integers(40, 90))) for _ in range(120)]
    outs = [gpu.nn_batch(spec, v, Q, C, precision="float32")[:2] for v in ("base", "ea", "eapruned", "pruned_only")]
    for idx, dist in outs[1:]:
        assert np.array_equal(idx, outs[0][0]) and np.array_equal(dist, outs[0][1])
    r = eko.nn(spec, "eapruned", Q, C)
    assert all(rel_ok(a, b) for a, b in zip(outs[0][1], r["nn_distance"]))
    # dense equal lengths take the LB_Keogh path: same answers as the full FP32 scan
    Qd = np.stack([walk(rng, 128) for _ in range(8)])
    Cd = np.stack([walk(rng, 128) for _ in range(300)])
    a = gpu.nn_batch(spec, "eapruned", Qd, Cd, precision="float32")[:2]
    b = gpu.nn_batch(spec, "base", Qd, Cd, precision="float32")[:2]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("kind", ["dtw", "cdtw", "wdtw", "erp", "msm", "twe"])
def test_fp32_pairwise(gpu, rng, kind):
    spec = random_spec(gpu, kind, rng, 96, "squared")
    X = np.stack([walk(rng, 96) for _ in range(24)])
    D, _ = gpu.pairwise(spec, X, precision="float32")
    R, _ = eko.pairwise(spec, X)
    assert np.array_equal(D, D.T) and not np.diag(D).any()
    bad = [(i, j, D[i, j], R[i, j]) for i in range(24) for j in range(24) if not rel_ok(D[i, j], R[i, j])]
    assert not bad, bad[:6]


@pytest.mark.parametrize("kind", ["dtw", "msm"])
def test_fp32_long_series_strip_engine(gpu, rng, kind):
    """More than 512 columns: the strip engine in FP32."""
    spec = gpu.DistanceSpec(kind="dtw") if kind == "dtw" else gpu.DistanceSpec(kind="msm", msm_c=0.5)
    pairs = [(walk(rng, int(rng.integers(520, 900))), walk(rng, int(rng.integers(520, 900)))) for _ in range(4)]
    got, _ = gpu.distance_batch(spec, "base", pairs, precision="float32")
    for (a, b), g in zip(pairs, got):
        assert rel_ok(g, eko.distance(spec, "base", a, b)[0])


def test_fp32_rejected_where_unsupported(gpu, rng):
    spec = gpu.DistanceSpec(kind="cdtw", window=3)
    with pytest.raises(gpu.SpecError, match="float64 only"):
        gpu.subsequence_search(walk(rng, 16), walk(rng, 200),
                               gpu.SearchConfig(spec=spec, precision="float32"))
