"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
golden fixtures from the live reference.  Bit-exact FP64 costs, identical 1-NN
indices / labels / +inf outcomes, lowest-index ties.

Mirrors the reference's backend-parity sweep (pkg/tests/test_backends.py:30-55),
its engine property tests (test_engines.py) and acceptance criteria 1-5.
"""

import json
import math

import numpy as np
import pytest

from conftest import FIG_S, FIG_T, load_golden, spec_from_dict
from oracle import eko

pytestmark = pytest.mark.gpu

VARIANTS = ("base", "ea", "eapruned", "pruned_only")


def same(a, b):
    return (a == b) or (math.isinf(a) and math.isinf(b) and (a > 0) == (b > 0))


def test_golden_pairs_gpu(gpu):
    g = load_golden("pairs.npz")
    specs = [spec_from_dict(d) for d in json.loads(str(g["specs"]))]
    ser, off, ln = g["series"], g["series_off"], g["series_len"]
    get = lambda k: ser[off[k]: off[k] + ln[k]]
    # group rows by (spec, variant) so each group is one batched GPU call
    bad = []
    keys = sorted(set(zip(g["spec_idx"].tolist(), g["variant"].tolist())))
    for si, vi in keys:
        rows = np.where((g["spec_idx"] == si) & (g["variant"] == vi))[0]
        pairs = [(get(g["a"][k]), get(g["b"][k])) for k in rows]
        costs, cells = gpu.distance_batch(specs[si], VARIANTS[vi], pairs, cutoffs=g["cutoff"][rows])
        for k, c, n in zip(rows, costs, cells):
            if not same(c, g["cost"][k]):
                bad.append((specs[si].kind, VARIANTS[vi], g["cutoff"][k], c, g["cost"][k]))
            if n != g["cells"][k]:  # EngineResult equality: the reference's own cell counts
                bad.append(("cells", specs[si].kind, VARIANTS[vi], g["cutoff"][k], int(n), int(g["cells"][k])))
    assert not bad, bad[:10]


@pytest.mark.parametrize("kind", ["dtw", "cdtw", "wdtw", "erp", "msm", "twe"])
def test_reference_cells_long_pairs(gpu, rng, kind):
    """cells_computed of ea / eapruned / pruned_only equal the reference's (oracle, which
    replays the reference's row stages) on pairs up to 300 points, every cutoff regime."""
    bad = []
    for mode in ("squared", "absolute"):
        spec = random_spec(gpu, kind, rng, 300, mode)
        pairs, cuts, want = [], [], []
        for _ in range(6):
            n1, n2 = int(rng.integers(150, 301)), int(rng.integers(150, 301))
            a, b = np.cumsum(rng.normal(0, 1, n1)), np.cumsum(rng.normal(0, 1, n2))
            exact = eko.distance(spec, "base", a, b)[0]
            for f in (np.inf, 1.02, 1.0, 0.97, 0.5):
                c = exact * f if np.isfinite(exact) else f
                pairs.append((a, b))
                cuts.append(c)
        for variant in ("ea", "eapruned", "pruned_only"):
            costs, cells = gpu.distance_batch(spec, variant, pairs, cutoffs=cuts)
            for (a, b), c, got_c, got_n in zip(pairs, cuts, costs, cells):
                ref = eko.distance(spec, variant, a, b, cutoff=c)
                if not (same(got_c, ref[0]) and got_n == ref[1]):
                    bad.append((kind, mode, variant, c, got_c, ref[0], int(got_n), int(ref[1])))
    assert not bad, bad[:6]


def random_spec(ekb, kind, rng, maxlen, mode):
    if kind == "dtw":
        return ekb.DistanceSpec(kind="dtw", cost_mode=mode)
    if kind == "cdtw":
        return ekb.DistanceSpec(kind="cdtw", window=int(rng.integers(0, maxlen + 1)), cost_mode=mode)
    if kind == "wdtw":
        return ekb.DistanceSpec(kind="wdtw", wdtw_g=float(rng.uniform(0.0, 0.6)), cost_mode=mode)
    if kind == "erp":
        return ekb.DistanceSpec(kind="erp", window=int(rng.integers(0, maxlen + 1)),
                                erp_gap=float(rng.uniform(-1.0, 1.0)), cost_mode=mode)
    if kind == "msm":
        return ekb.DistanceSpec(kind="msm", msm_c=float(rng.uniform(0.0, 2.0)), cost_mode=mode)
    return ekb.DistanceSpec(kind="twe", twe_nu=float(rng.uniform(0.0, 1.0)),
                            twe_lambda=float(rng.uniform(0.0, 2.0)), cost_mode=mode)


@pytest.mark.parametrize("kind", ["dtw", "cdtw", "wdtw", "erp", "msm", "twe"])
@pytest.mark.parametrize("mode", ["squared", "absolute"])
def test_random_sweep_vs_oracle(gpu, kind, mode):
    """Lengths 1..300 (both engines, every band shape), cutoffs {inf,1.05,1,0.95,0.3}x exact."""
    rng = np.random.default_rng(hash((kind, mode)) % 2**32)
    bad = []
    for trial in range(60):
        hi = 48 if trial < 40 else 300
        la, lb = int(rng.integers(1, hi)), int(rng.integers(1, hi))
        spec = random_spec(gpu, kind, rng, max(la, lb), mode)
        a = np.cumsum(rng.normal(0, 1, la))
        b = np.cumsum(rng.normal(0, 1, lb))
        exact = eko.distance(spec, "base", a, b)[0]
        cuts = [math.inf]
        if math.isfinite(exact) and exact > 0:
            cuts += [exact * f for f in (1.05, 1.0, 0.95, 0.3)]
        for v in VARIANTS:
            costs, _ = gpu.distance_batch(spec, v, [(a, b)] * len(cuts), cutoffs=cuts)
            for co, c in zip(cuts, costs):
                want = eko.distance(spec, v, a, b, co)[0]
                if not same(c, want):
                    bad.append((la, lb, spec.window, v, co, c, want))
    assert not bad, bad[:8]


def test_fig1_and_fig2b(gpu):
    dtw = gpu.DistanceSpec(kind="dtw")
    for v in VARIANTS:
        assert gpu.distance(dtw, v, FIG_S, FIG_T).cost == 9.0
    assert gpu.distance(dtw, "base", FIG_S, FIG_T) == (9.0, 36)
    assert math.isinf(gpu.distance(dtw, "eapruned", FIG_S, FIG_T, cutoff=6.0).cost)
    assert gpu.distance(dtw, "eapruned", FIG_S, FIG_T, cutoff=9.0).cost == 9.0
    assert math.isinf(gpu.distance(dtw, "ea", FIG_S, FIG_T, cutoff=6.0).cost)
    spec = gpu.DistanceSpec(kind="cdtw", window=1)
    for v in VARIANTS:
        r = gpu.distance(spec, v, FIG_S, [1.0, 2, 3, 4, 5, 6, 7, 8])
        assert math.isinf(r.cost) and r.cells_computed == 0


def test_nan_and_negative_zero_cutoffs(gpu, rng):
    spec = gpu.DistanceSpec(kind="cdtw", window=3)
    a, b = rng.normal(0, 1, 12), rng.normal(0, 1, 9)
    for v in ("ea", "eapruned"):
        for co in (math.nan, -0.0, 0.0, -1.0, -math.inf):
            got = gpu.distance(spec, v, a, b, cutoff=co).cost
            want = eko.distance(spec, v, a, b, co)[0]
            assert same(got, want), (v, co, got, want)
    z = np.zeros(7)
    for v in ("ea", "eapruned"):
        assert gpu.distance(spec, v, z, z, cutoff=-0.0).cost == eko.distance(spec, v, z, z, -0.0)[0]


def test_identical_series_zero_all_kinds(gpu, rng):
    s = rng.uniform(-4, 4, 12)
    for kind in gpu.KINDS:
        spec = random_spec(gpu, kind, rng, 12, "squared")
        for v in VARIANTS:
            assert gpu.distance(spec, v, s, s).cost == 0.0


def test_golden_nn_gpu(gpu):
    g = load_golden("nn.npz")
    specs = [spec_from_dict(d) for d in json.loads(str(g["specs"]))]
    for k, spec in enumerate(specs):
        train = gpu.LabeledDataset("train", tuple((int(a), b) for a, b in zip(g[f"y{k}"], g[f"X{k}"])))
        test = gpu.LabeledDataset("test", tuple((int(a), b) for a, b in zip(g[f"qy{k}"], g[f"Q{k}"])))
        for variant in VARIANTS:
            recs = gpu.classify_1nn(train, test, gpu.SearchConfig(spec=spec, variant=variant))
            assert [r.nn_index for r in recs] == g[f"idx{k}"].tolist(), (spec, variant)
            assert [r.nn_distance for r in recs] == g[f"dist{k}"].tolist(), (spec, variant)
            assert [r.predicted for r in recs] == g[f"pred{k}"].tolist(), (spec, variant)
    idx = gpu.nn_batch(gpu.DistanceSpec(kind="dtw"), "eapruned", g["tie_Q"], g["tie_X"])[0]
    assert np.array_equal(idx, g["tie_idx"])


def test_nn_ragged_and_unequal_lengths(gpu, rng):
    q = [np.cumsum(rng.normal(0, 1, n)) for n in (20, 31, 17)]
    c = [np.cumsum(rng.normal(0, 1, n)) for n in (20, 14, 26, 20, 40, 19)]
    for spec in (gpu.DistanceSpec(kind="dtw"), gpu.DistanceSpec(kind="cdtw", window=7),
                 gpu.DistanceSpec(kind="wdtw", wdtw_g=0.1), gpu.DistanceSpec(kind="erp", window=9, erp_gap=0.5),
                 gpu.DistanceSpec(kind="msm", msm_c=0.5), gpu.DistanceSpec(kind="twe", twe_nu=0.1, twe_lambda=1.0)):
        idx, dist = gpu.nn_batch(spec, "eapruned", q, c)[:2]
        r = eko.nn(spec, "eapruned", q, c, threads=2)
        assert np.array_equal(idx, r["nn_index"]), spec
        assert np.array_equal(dist, r["nn_distance"]), spec


def test_nn_search_single_and_self_match(gpu, rng):
    dtw = gpu.DistanceSpec(kind="dtw")
    q = rng.normal(0, 1, 16)
    d, i, st = gpu.nn_search(q, [q, rng.normal(0, 1, 16)], gpu.SearchConfig(spec=dtw))
    assert (d, i) == (0.0, 0)
    assert st.computed + st.abandoned == 2
    with pytest.raises(gpu.SearchError):
        gpu.nn_search([1.0, 2.0], [], gpu.SearchConfig(spec=dtw))


def test_golden_pairwise_gpu(gpu):
    g = load_golden("pairwise.npz")
    D, cells = gpu.pairwise(gpu.DistanceSpec(kind="wdtw", wdtw_g=0.05), g["X"])
    assert np.array_equal(D, g["D_wdtw"])
    assert cells > 0
    D, _ = gpu.pairwise(gpu.DistanceSpec(kind="erp", window=4, erp_gap=0.0), g["X"])
    assert np.array_equal(D, g["D_erp"])


def test_pairwise_all_kinds_vs_oracle(gpu, rng):
    X = [np.cumsum(rng.normal(0, 1, n)) for n in rng.integers(5, 60, size=14)]
    for kind in gpu.KINDS:
        for mode in ("squared", "absolute"):
            spec = random_spec(gpu, kind, rng, 40, mode)
            D, _ = gpu.pairwise(spec, X)
            Do, _ = eko.pairwise(spec, X, threads=2)
            assert np.array_equal(D, Do), (spec,)


def test_golden_subseq_gpu(gpu):
    g = load_golden("subseq.npz")
    for k, (kind, w, norm) in enumerate(json.loads(str(g["cases"]))):
        spec = gpu.DistanceSpec(kind=kind, window=w)
        for variant in VARIANTS:
            off, d, st = gpu.subsequence_search(g["q"], g["ref"],
                                                gpu.SearchConfig(spec=spec, variant=variant, normalize=norm))
            assert (off, d) == (g["off"][k], g["dist"][k]), (kind, w, norm, variant)
            assert st.computed + st.abandoned == len(g["ref"]) - len(g["q"]) + 1


def test_subseq_edge_cases(gpu):
    dtw = gpu.DistanceSpec(kind="dtw")
    assert gpu.subsequence_search([1.0, 2.0], [0.0, 1.0, 2.0, 3.0], gpu.SearchConfig(spec=dtw, variant="base"))[:2] \
        == (1, 0.0)
    assert gpu.subsequence_search([7.0, 7.0], [7.0] * 4, gpu.SearchConfig(spec=dtw, variant="base"))[:2] == (0, 0.0)
    with pytest.raises(gpu.DimensionError):
        gpu.subsequence_search([1.0, 2.0, 3.0], [1.0, 2.0], gpu.SearchConfig(spec=dtw))
    with pytest.raises(gpu.SpecError):
        gpu.subsequence_search([1.0, 2.0], [1.0, 2.0, 3.0], gpu.SearchConfig(spec=gpu.DistanceSpec("msm", msm_c=1.0)))


def test_subseq_normalized_planted_copy(gpu, rng):
    # pkg/tests/test_search.py:173-181
    q = np.cumsum(rng.normal(0, 1, 24))
    ref = rng.normal(50.0, 0.25, 200)
    ref[130:154] = 3.5 * q + 20.0
    off, d, _ = gpu.subsequence_search(q, ref, gpu.SearchConfig(spec=gpu.DistanceSpec(kind="dtw"), normalize=True))
    assert off == 130 and d < 1e-12


def test_subseq_vs_oracle_random(gpu, rng):
    for lq, n, w, norm in ((64, 3000, 6, True), (100, 2500, None, True), (33, 1500, 3, False), (200, 4000, 10, True)):
        q = np.cumsum(rng.normal(0, 1, lq))
        ref = np.cumsum(rng.normal(0, 1, n))
        spec = gpu.DistanceSpec(kind="dtw" if w is None else "cdtw", window=w)
        got = gpu.subsequence_search(q, ref, gpu.SearchConfig(spec=spec, normalize=norm))[:2]
        want = eko.subsequence(spec, "eapruned", q, ref, norm, chunk=256, threads=4)[:2]
        assert got == want, (lq, n, w, norm)


@pytest.mark.parametrize("lq,w,norm,mode", [(1, 0, False, "squared"), (7, 2, True, "squared"),
                                            (129, 9, True, "squared"), (300, 31, True, "absolute"),
                                            (64, None, True, "squared"), (200, 40, False, "absolute")])
def test_subseq_profile_every_window(gpu, rng, lq, w, norm, mode):
    """Every window's distance (not just the best) matches the oracle bit for bit;
    the stream holds flat runs (all-zeros z-normalised windows) and spikes."""
    ref = np.cumsum(rng.normal(0, 1, 3000))
    ref[500:900] = 4.25          # flat run: std < 1e-12 windows
    ref[1500:1520] *= 1e6        # large dynamic range
    ref[2000:2300] = rng.normal(0, 1e-7, 300)
    q = np.cumsum(rng.normal(0, 1, lq))
    spec = gpu.DistanceSpec(kind="dtw" if w is None else "cdtw", window=w, cost_mode=mode)
    got = gpu.subsequence_profile(q, ref, spec, normalize=norm)
    want = eko.subsequence_profile(spec, q, ref, norm, threads=4)
    assert got.shape == want.shape
    assert np.array_equal(got, want), int(np.flatnonzero(got != want)[0])


@pytest.mark.parametrize("kind,window,mode", [("cdtw", 12, "squared"), ("dtw", None, "squared"),
                                              ("cdtw", 7, "absolute")])
def test_nn_lb_filter_scale(gpu, kind, window, mode):
    """Dense dtw/cdtw 1-NN takes the LB_Keogh pre-filter path: results must not change."""
    from paper_2102_05221_b200 import datagen

    C, cl, protos = datagen.warped_prototypes(1024, 128, 8, 0.1, 77)
    Q, ql, _ = datagen.warped_prototypes(48, 128, 8, 0.1, 78, protos=protos)
    Q[5] = C[300]  # exact duplicate -> distance 0, lowest index must win
    C[301] = C[300]
    spec = gpu.DistanceSpec(kind=kind, window=window, cost_mode=mode)
    idx, dist, cells, comp, ab = gpu.nn_batch(spec, "eapruned", Q, C)
    r = eko.nn(spec, "eapruned", Q, C, threads=4)
    assert np.array_equal(idx, r["nn_index"])
    assert np.array_equal(dist, r["nn_distance"])
    assert idx[5] == 300 and dist[5] == 0.0
    assert np.all(comp + ab == len(C))


@pytest.mark.parametrize("kind", ["msm", "twe", "dtw", "wdtw"])
def test_nn_guarded_band(gpu, kind):
    """Unconstrained series longer than a P=8 band: phase B runs the guarded band
    (ek_kernels.cuh E_GDIAG8) and must return the oracle's answer exactly."""
    from paper_2102_05221_b200 import datagen

    C, cl, protos = datagen.warped_prototypes(300, 400, 6, 0.2, 91)
    Q, ql, _ = datagen.warped_prototypes(8, 400, 6, 0.2, 92, protos=protos)
    params = {"msm": dict(msm_c=1.0), "twe": dict(twe_nu=0.001, twe_lambda=1.0), "dtw": {}, "wdtw": dict(wdtw_g=0.05)}
    spec = gpu.DistanceSpec(kind=kind, **params[kind])
    for variant in ("eapruned", "ea"):
        idx, dist = gpu.nn_batch(spec, variant, Q, C)[:2]
        r = eko.nn(spec, variant, Q, C, threads=4)
        assert np.array_equal(idx, r["nn_index"]), (kind, variant)
        assert np.array_equal(dist, r["nn_distance"]), (kind, variant)


@pytest.mark.parametrize("kind", ["msm", "dtw"])
def test_nn_guard_overflow_redo(gpu, rng, kind):
    """Near-constant series keep every cell under the cutoff, so the guarded band
    overflows and k_nn_fix redoes the pairs: still the oracle's answer."""
    C = rng.normal(0.0, 1e-3, size=(40, 300))
    Q = rng.normal(0.0, 1e-3, size=(3, 300))
    C[7] = Q[1]
    spec = gpu.DistanceSpec(kind=kind, msm_c=1.0) if kind == "msm" else gpu.DistanceSpec(kind=kind)
    idx, dist = gpu.nn_batch(spec, "eapruned", Q, C)[:2]
    r = eko.nn(spec, "eapruned", Q, C, threads=4)
    assert np.array_equal(idx, r["nn_index"]) and np.array_equal(dist, r["nn_distance"])
    assert idx[1] == 7 and dist[1] == 0.0


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_inputs_raise(gpu, rng, bad):
    """as_series' contract (series.py:19-28) for the dense in-place path, where the
    library checks the uploaded copy: ValueError with the reference's message."""
    Q = rng.normal(size=(3, 40))
    C = rng.normal(size=(9, 40))
    C[4, 17] = bad
    spec = gpu.DistanceSpec(kind="cdtw", window=4)
    with pytest.raises(ValueError, match="must all be finite"):
        gpu.nn_batch(spec, "eapruned", Q, C)
    with pytest.raises(ValueError, match="must all be finite"):
        gpu.pairwise(spec, C)
    Qb = Q.copy()
    Qb[1, 3] = bad
    with pytest.raises(ValueError, match="must all be finite"):
        gpu.nn_batch(spec, "eapruned", Qb, C[:4])
    ref = rng.normal(size=200)
    ref[50] = bad
    with pytest.raises(ValueError, match="must all be finite"):
        gpu.subsequence_search(Q[0], ref, gpu.SearchConfig(spec=spec))
    # a long stream is validated on the device only (as_series(finite_on_device=True))
    long_ref = rng.normal(size=6000)
    long_ref[4321] = bad
    with pytest.raises(ValueError, match="must all be finite"):
        gpu.subsequence_search(Q[0], long_ref, gpu.SearchConfig(spec=spec))
    with pytest.raises(ValueError, match="must all be finite"):
        gpu.subsequence_profile(Q[0], long_ref, spec)
    # the library stays usable afterwards
    idx = gpu.nn_batch(spec, "eapruned", Q, C[:4])[0]
    assert idx.shape == (3,)


def _workload_rows(wl, nq, seed_shift=0):
    from paper_2102_05221_b200 import datagen

    C, cl, protos = datagen.warped_prototypes(wl.n_candidates, wl.length, wl.classes, wl.sigma, wl.seed)
    Q, ql, _ = datagen.warped_prototypes(nq, wl.length, wl.classes, wl.sigma, wl.seed + 1 + seed_shift,
                                         protos=protos)
    return Q, C


@pytest.mark.parametrize("which", ["c2", "c4m", "c4t"])
def test_benchmark_shapes_vs_oracle(gpu, which):
    """The BASELINE configurations at full candidate count and length, on a query subset
    the oracle finishes in seconds: nn indices and distances identical."""
    from paper_2102_05221_b200 import datagen

    wl = datagen.C2 if which == "c2" else datagen.C4
    nq = 32 if which == "c2" else 8
    Q, C = _workload_rows(wl, nq)
    spec = {"c2": gpu.DistanceSpec(kind="cdtw", window=51),
            "c4m": gpu.DistanceSpec(kind="msm", msm_c=1.0),
            "c4t": gpu.DistanceSpec(kind="twe", twe_nu=0.001, twe_lambda=1.0)}[which]
    idx, dist = gpu.nn_batch(spec, "eapruned", Q, C)[:2]
    r = eko.nn(spec, "eapruned", Q, C, threads=16)
    assert np.array_equal(idx, r["nn_index"]) and np.array_equal(dist, r["nn_distance"])


def test_c2_full_size_properties(gpu, rng):
    """Full C2 size (256 x 4096 x 512): results are invariant under any candidate order
    (indices map back through the permutation) and equal to base-variant distances."""
    from paper_2102_05221_b200 import datagen

    Q, _, C, _ = datagen.C2.make()
    spec = gpu.DistanceSpec(kind="cdtw", window=51)
    idx, dist = gpu.nn_batch(spec, "eapruned", Q, C)[:2]
    perm = rng.permutation(len(C))
    idx_p, dist_p = gpu.nn_batch(spec, "eapruned", Q, np.ascontiguousarray(C[perm]))[:2]
    assert np.array_equal(dist, dist_p)
    assert np.array_equal(perm[idx_p], idx)  # no exact ties in this data
    # every reported distance is the exact (base) distance of that pair
    pairs = [(Q[k], C[idx[k]]) for k in range(0, len(Q), 16)]
    base, _ = gpu.distance_batch(spec, "base", pairs)
    assert np.array_equal(base, dist[::16])


def test_subseq_long_stream_vs_oracle(gpu):
    """C5 shape (query 1024, w=51, z-normalised) on a 2^15-point stream: best window and
    distance identical to the oracle; the planted copy is found at distance ~0."""
    from paper_2102_05221_b200 import datagen

    stream, q = datagen.subsequence_workload(stream_len=1 << 15, query_len=1024, seed=4242)
    spec = gpu.DistanceSpec(kind="cdtw", window=51)
    got = gpu.subsequence_search(q, stream, gpu.SearchConfig(spec=spec, variant="eapruned", normalize=True))[:2]
    want = eko.subsequence(spec, "eapruned", q, stream, True, chunk=2048, threads=16)[:2]
    assert got == want


@pytest.mark.parametrize("kind", ["dtw", "wdtw", "erp", "msm", "twe", "cdtw"])
def test_long_series_strip_engine(gpu, rng, kind):
    """Series longer than one 512-column strip (up to 1300 points): unconstrained or
    wide-band pairs run the strip engine (ek_stripe.cuh strip_pair) -- costs equal the
    oracle's for every variant and cutoff regime, cells for base."""
    params = {"dtw": {}, "cdtw": dict(window=700), "wdtw": dict(wdtw_g=0.02), "erp": dict(window=900, erp_gap=0.1),
              "msm": dict(msm_c=0.5), "twe": dict(twe_nu=0.001, twe_lambda=1.0)}[kind]
    spec = gpu.DistanceSpec(kind=kind, **params)
    pairs, cuts = [], []
    for _ in range(4):
        n1, n2 = int(rng.integers(520, 1300)), int(rng.integers(520, 1300))
        a, b = np.cumsum(rng.normal(0, 1, n1)), np.cumsum(rng.normal(0, 1, n2))
        ex = eko.distance(spec, "base", a, b)[0]
        for f in (np.inf, 1.01, 0.99):
            pairs.append((a, b))
            cuts.append(ex * f if np.isfinite(ex) else f)
    bad = []
    for variant in ("base", "ea", "eapruned", "pruned_only"):
        costs, cells = gpu.distance_batch(spec, variant, pairs, cutoffs=cuts)
        for (a, b), c, got, n in zip(pairs, cuts, costs, cells):
            ref = eko.distance(spec, variant, a, b, cutoff=c)
            if not same(got, ref[0]) or (variant == "base" and n != ref[1]):
                bad.append((variant, c, got, ref[0], int(n), int(ref[1])))
    assert not bad, bad[:5]


@pytest.mark.parametrize("kind", ["dtw", "msm"])
def test_long_series_nn_and_pairwise(gpu, kind):
    """1-NN and all-pairs on 1000-point series (strip engine; guarded band + strip redo
    for the cutoff variants) against the oracle."""
    from paper_2102_05221_b200 import datagen

    C, cl, protos = datagen.warped_prototypes(40, 1000, 4, 0.2, 71)
    Q, ql, _ = datagen.warped_prototypes(3, 1000, 4, 0.2, 72, protos=protos)
    spec = gpu.DistanceSpec(kind=kind, msm_c=1.0) if kind == "msm" else gpu.DistanceSpec(kind=kind)
    for variant in ("eapruned", "base"):
        idx, dist = gpu.nn_batch(spec, variant, Q, C)[:2]
        r = eko.nn(spec, variant, Q, C, threads=16)
        assert np.array_equal(idx, r["nn_index"]) and np.array_equal(dist, r["nn_distance"]), variant
    D, _ = gpu.pairwise(spec, C[:8])
    Do, _ = eko.pairwise(spec, C[:8], threads=16)
    assert np.array_equal(D, Do)


@pytest.mark.parametrize("offset,scale", [(1e7, 1e-3), (1e4, 1.0), (0.0, 1e-9), (-3e5, 50.0)])
def test_subseq_lb_statistics_regimes(gpu, rng, offset, scale):
    """The LB pass's prefix-sum statistics across numeric regimes: huge offsets with a
    tiny spread (the bound gives up and the DP decides), near-zero-std windows, wide
    walks -- best window and distance equal the oracle's (z-normalised search)."""
    n, lq = 6000, 200
    stream = offset + scale * np.cumsum(rng.normal(0, 1, n))
    stream[2000:2300] = offset  # a flat run: std < 1e-12 windows
    q = stream[4100:4100 + lq] + scale * 0.01 * rng.normal(0, 1, lq)
    for kind, w in (("cdtw", 10), ("dtw", None)):
        spec = gpu.DistanceSpec(kind=kind, window=w)
        for variant in ("eapruned", "ea"):
            got = gpu.subsequence_search(q, stream, gpu.SearchConfig(spec=spec, variant=variant, normalize=True))[:2]
            want = eko.subsequence(spec, "eapruned", q, stream, True, chunk=500, threads=16)[:2]
            assert got == want, (kind, variant, got, want)


@pytest.mark.parametrize("length,window", [(1, 0), (7, 3), (100, 0), (100, 1), (128, 51), (512, 51), (300, 299),
                                           (300, 5000), (1000, 127), (7000, 64), (7000, 3000)])
def test_build_envelopes_match_host(gpu, rng, length, window):
    """Batched GPU envelopes (k_envelope, exact tables; shared memory and, past 6144
    points, global scratch rows) equal build_envelope's values."""
    from paper_2102_05221_b200 import lower_bounds as lbm

    X = np.cumsum(rng.normal(0, 1, (5, length)), axis=1)
    X[1] = np.round(X[1])  # ties
    got = lbm.build_envelopes(X, window)
    for k in range(len(X)):
        want = lbm.build_envelope(X[k], window)
        assert np.array_equal(got[k].upper, want.upper), (k, length, window)
        assert np.array_equal(got[k].lower, want.lower), (k, length, window)


def test_nn_lb_long_series_scratch_envelope(gpu):
    """cdtw 1-NN on 13000-point series: the LB envelopes exceed shared memory and are
    built in global scratch rows; the answer must equal the oracle's."""
    from paper_2102_05221_b200 import datagen

    C, cl, protos = datagen.warped_prototypes(7, 13000, 3, 0.2, 61)
    Q, ql, _ = datagen.warped_prototypes(2, 13000, 3, 0.2, 62, protos=protos)
    spec = gpu.DistanceSpec(kind="cdtw", window=20)
    idx, dist = gpu.nn_batch(spec, "eapruned", Q, C)[:2]
    r = eko.nn(spec, "eapruned", Q, C, threads=16)
    assert np.array_equal(idx, r["nn_index"]) and np.array_equal(dist, r["nn_distance"])


@pytest.mark.parametrize("where", [0, 37, 63])
def test_nonfinite_in_any_upload_chunk(gpu, rng, where):
    """The candidates go up in chunks (ek_nn); a non-finite value in any chunk raises."""
    Q = rng.normal(size=(2, 24))
    C = rng.normal(size=(64, 24))
    C[where, 5] = np.nan
    spec = gpu.DistanceSpec(kind="cdtw", window=3)
    with pytest.raises(ValueError, match="must all be finite"):
        gpu.nn_batch(spec, "eapruned", Q, C)


def test_nn_lb_path_beyond_rank_limit(gpu, rng):
    """More than 16384 candidates: the LB path keeps the keys but skips the ranking
    (identity order); answers still equal the oracle's, ties to the lowest index."""
    L, n = 24, 16500
    C = np.cumsum(rng.normal(size=(n, L)), axis=1)
    Q = C[[5, 9000, 16400]] + rng.normal(0, 1e-3, size=(3, L))
    C[12000] = C[9000]  # an exact duplicate of a near-neighbour: the lower index must win
    spec = gpu.DistanceSpec(kind="cdtw", window=2)
    idx, dist = gpu.nn_batch(spec, "eapruned", Q, C)[:2]
    r = eko.nn(spec, "eapruned", Q, C, threads=16)
    assert np.array_equal(idx, r["nn_index"]) and np.array_equal(dist, r["nn_distance"])
    assert idx[1] == 9000


@pytest.mark.parametrize("kind,window,n", [("erp", 25, 33), ("cdtw", 12, 40), ("cdtw", 29, 17), ("erp", 3, 8)])
def test_pairwise_half_warp_pairs(gpu, rng, kind, window, n):
    """Bands of <= 64 diagonal slots run two pairs per warp in lockstep (E_DIAG4H): equal
    lengths (the lockstep path), an odd number of pairs (a lone last pair), and a ragged
    set (pairs of different shapes run one after the other); bit-exact with the oracle."""
    spec = (gpu.DistanceSpec(kind="erp", window=window, erp_gap=0.3) if kind == "erp"
            else gpu.DistanceSpec(kind="cdtw", window=window))
    X = np.cumsum(rng.normal(size=(n, 90)), axis=1)
    D, cells = gpu.pairwise(spec, X)
    Do, cells_o = eko.pairwise(spec, X, threads=8)
    assert np.array_equal(D, Do)
    Xr = [np.cumsum(rng.normal(size=int(m))) for m in rng.integers(60, 91, size=n)]
    D, _ = gpu.pairwise(spec, Xr)
    Do, _ = eko.pairwise(spec, Xr, threads=8)
    assert np.array_equal(D, Do)


@pytest.mark.parametrize("kind", ["wdtw", "dtw", "twe", "msm", "erp"])
def test_pairwise_half_warp_stripe(gpu, rng, kind):
    """Unbanded all-pairs of 129..256 columns run two pairs per warp on the S=16 row stripe
    (E_STR16H): dense (lockstep) and ragged (one pair at a time) sets, bit-exact."""
    spec = {"wdtw": gpu.DistanceSpec(kind="wdtw", wdtw_g=0.05), "dtw": gpu.DistanceSpec(kind="dtw"),
            "twe": gpu.DistanceSpec(kind="twe", twe_nu=0.01, twe_lambda=0.5),
            "msm": gpu.DistanceSpec(kind="msm", msm_c=0.5),
            "erp": gpu.DistanceSpec(kind="erp", window=400, erp_gap=0.1)}[kind]
    X = np.cumsum(rng.normal(size=(9, 200)), axis=1)
    D, _ = gpu.pairwise(spec, X)
    Do, _ = eko.pairwise(spec, X, threads=8)
    assert np.array_equal(D, Do)
    Xr = [np.cumsum(rng.normal(size=int(m))) for m in rng.integers(150, 257, size=7)]
    D, _ = gpu.pairwise(spec, Xr)
    Do, _ = eko.pairwise(spec, Xr, threads=8)
    assert np.array_equal(D, Do)


@pytest.mark.parametrize("kind,window", [("cdtw", 5), ("dtw", None)])
def test_nn_candidate_halves_ties_and_seeding(gpu, rng, kind, window, monkeypatch):
    """ek_nn from host arrays splits a large LB-path search into two candidate halves (the
    second seeded with the first's answers): an exact duplicate across the halves resolves
    to the lower index, a neighbour only in the second half is found, and everything equals
    the oracle's serial scan."""
    L, n = 40, 4096
    C = np.cumsum(rng.normal(size=(n, L)), axis=1)
    C[3000] = C[100]  # duplicate across the halves: index 100 must win
    Q = np.stack([C[100] + 1e-3, C[3500] + 1e-3, C[2047] + 2e-3, rng.normal(size=L).cumsum()])
    spec = gpu.DistanceSpec(kind=kind, window=window)
    monkeypatch.setenv("EKB_NN_SPLIT", "2")  # read per call by the library (default 1: measured slower on C2)
    for variant in ("eapruned", "ea"):
        idx, dist = gpu.nn_batch(spec, variant, Q, C)[:2]
        r = eko.nn(spec, variant, Q, C, threads=16)
        assert np.array_equal(idx, r["nn_index"]) and np.array_equal(dist, r["nn_distance"]), (idx, r["nn_index"])
        assert idx[0] == 100 and idx[1] == 3500


@pytest.mark.parametrize("lq,window,norm", [(600, None, True), (1024, None, False), (700, 300, True),
                                             (513, None, True)])
def test_subseq_long_query_strip_engines(gpu, rng, lq, window, norm):
    """Queries longer than one 512-column row stripe: unbanded DTW and wide-band CDTW run the
    strip engines inside the subsequence kernel (search.py:163-215 takes any length).  The
    best window equals the oracle's; a planted copy is found."""
    stream = np.cumsum(rng.normal(size=lq + 1400))
    q = stream[901:901 + lq] + rng.normal(0, 1e-3, size=lq)
    spec = gpu.DistanceSpec(kind="cdtw" if window is not None else "dtw", window=window)
    got = gpu.subsequence_search(q, stream, gpu.SearchConfig(spec=spec, variant="eapruned", normalize=norm))[:2]
    want = eko.subsequence(spec, "eapruned", q, stream, norm, chunk=256, threads=16)[:2]
    assert got == want and got[0] == 901, (got, want)


def test_subseq_profile_long_query(gpu, rng):
    """Every window's exact distance for a 600-point unbanded DTW query (strip engine)."""
    stream = np.cumsum(rng.normal(size=760))
    q = np.cumsum(rng.normal(size=600))
    spec = gpu.DistanceSpec(kind="dtw")
    prof = gpu.subsequence_profile(q, stream, spec, normalize=True)
    want = eko.subsequence_profile(spec, q, stream, True, threads=16)
    assert np.array_equal(np.asarray(prof), want)
