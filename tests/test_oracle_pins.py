"""Pin the CPU oracle (oracle/ek_oracle.c) before trusting it as the GPU checker.

* against the golden fixtures recorded from the live reference (make_golden.py);
* against the reference's own known-answer tests (pkg/tests/test_engines.py,
  test_acceptance.py, test_kernels.py);
* numpy's pairwise-sum / z-normalisation order (series.py:118-131), which the
  subsequence kernel reproduces on the GPU.
"""

import json
import math

import numpy as np
import pytest

from conftest import FIG_S, FIG_T, load_golden, spec_from_dict
from oracle import eko
from paper_2102_05221_b200 import DistanceSpec

VARIANTS = ("base", "ea", "eapruned", "pruned_only")
DTW = DistanceSpec(kind="dtw")


def test_golden_pairs_costs_and_cells():
    g = load_golden("pairs.npz")
    specs = [spec_from_dict(d) for d in json.loads(str(g["specs"]))]
    ser, off, ln = g["series"], g["series_off"], g["series_len"]
    bad = 0
    for k in range(len(g["cost"])):
        a = ser[off[g["a"][k]]: off[g["a"][k]] + ln[g["a"][k]]]
        b = ser[off[g["b"][k]]: off[g["b"][k]] + ln[g["b"][k]]]
        cost, cells = eko.distance(specs[g["spec_idx"][k]], VARIANTS[g["variant"][k]], a, b, g["cutoff"][k])
        want = g["cost"][k]
        same = (cost == want) or (math.isinf(cost) and math.isinf(want))
        bad += (not same) or cells != g["cells"][k]
    assert bad == 0


def test_fig1_golden_all_variants():
    # test_acceptance.py:44-48 / test_engines.py:22-25
    for v in VARIANTS:
        assert eko.distance(DTW, v, FIG_S, FIG_T)[0] == 9.0
    assert eko.distance(DTW, "base", FIG_S, FIG_T) == (9.0, 36)


def test_fig4_cell_counts():
    # test_acceptance.py:51-62
    c, n = eko.distance(DTW, "eapruned", FIG_S, FIG_T, 6.0)
    assert math.isinf(c) and abs(n - 20) <= 2
    c, n = eko.distance(DTW, "eapruned", FIG_S, FIG_T, 9.0)
    assert c == 9.0 and abs(n - 31) <= 2
    c, n = eko.distance(DTW, "ea", FIG_S, FIG_T, 6.0)
    assert math.isinf(c) and n == 30


def test_infeasible_window():
    # test_acceptance.py:65-71
    spec = DistanceSpec(kind="cdtw", window=1)
    for v in VARIANTS:
        c, n = eko.distance(spec, v, FIG_S, [1.0, 2, 3, 4, 5, 6, 7, 8])
        assert math.isinf(c) and n == 0


def test_wdtw_frozen_weight():
    # test_kernels.py:43-45
    assert abs(eko.wdtw_weight(0.1, 0, 100) - 0.0066928509242848554) < 1e-15
    assert eko.wdtw_table(0.3, 100)[50] == 0.5


def test_erp_border_prefix_through_engine():
    # test_kernels.py:119-124: border prefix 9, 10 -> d(([3,1]),([0,0])) via the left border
    spec = DistanceSpec(kind="erp", window=2, erp_gap=0.0)
    assert eko.distance(spec, "base", [3.0, 1.0], [3.0, 1.0])[0] == 0.0
    # against [0.0] with gap 0 every path costs the left-border prefix vborder(2) = 9 + 1
    assert eko.distance(spec, "base", [3.0, 1.0], [0.0])[0] == 10.0


def test_diag_ub_matches_squared_euclid(rng):
    # test_engines.py:177-185
    a, b = rng.uniform(-4, 4, 20), rng.uniform(-4, 4, 20)
    acc = 0.0
    for x, y in zip(a.tolist(), b.tolist()):
        acc += (x - y) * (x - y)
    assert eko.diagonal_upper_bound(DTW, a, b) == acc


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 127, 128, 129, 255, 256, 257, 500, 1000, 1023, 1024, 1025, 3000])
def test_numpy_pairwise_sum_order(n):
    rng = np.random.default_rng(n)
    for _ in range(20):
        a = rng.normal(0, 1, n) * 10.0 ** rng.uniform(-3, 3)
        assert eko.np_sum(a) == np.add.reduce(a)
        if n >= 2:
            m, s = a.mean(), a.std()
            want = np.zeros_like(a) if s < 1e-12 else (a - m) / s
            assert np.array_equal(eko.znormalize(a), want)


def test_golden_nn_fixtures():
    g = load_golden("nn.npz")
    specs = [spec_from_dict(d) for d in json.loads(str(g["specs"]))]
    for k, spec in enumerate(specs):
        r = eko.nn(spec, "eapruned", g[f"Q{k}"], g[f"X{k}"], threads=2)
        assert np.array_equal(r["nn_index"], g[f"idx{k}"])
        assert np.array_equal(r["nn_distance"], g[f"dist{k}"])
    r = eko.nn(DTW, "eapruned", g["tie_Q"], g["tie_X"], threads=2)
    assert np.array_equal(r["nn_index"], g["tie_idx"])


def test_golden_pairwise_fixtures():
    g = load_golden("pairwise.npz")
    D, _ = eko.pairwise(DistanceSpec(kind="wdtw", wdtw_g=0.05), g["X"], threads=2)
    assert np.array_equal(D, g["D_wdtw"])
    D, _ = eko.pairwise(DistanceSpec(kind="erp", window=4, erp_gap=0.0), g["X"], threads=2)
    assert np.array_equal(D, g["D_erp"])


def test_golden_subseq_fixtures():
    g = load_golden("subseq.npz")
    for k, (kind, w, norm) in enumerate(json.loads(str(g["cases"]))):
        spec = DistanceSpec(kind=kind, window=w)
        for chunk in (None, 97):
            off, d, _ = eko.subsequence(spec, "eapruned", g["q"], g["ref"], norm, chunk=chunk, threads=2)
            assert (off, d) == (g["off"][k], g["dist"][k])


def test_refdrive_glue_matches_the_live_reference():
    """The restated search loops around the reference's compiled kernel (oracle/refdrive.py,
    the bench's CPU arm) give the live reference's answers, for every lb mode."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import refpkg
    from oracle import refdrive

    ek = refpkg.load()
    if ek is None or not refdrive.available():
        pytest.skip("reference package / oracle/_ref not present (GPU box)")
    rng = np.random.default_rng(31)
    X = [np.cumsum(rng.normal(size=40)) for _ in range(25)] + [np.cumsum(rng.normal(size=33))]
    Q = [np.cumsum(rng.normal(size=40)) for _ in range(3)]
    for spec, refspec in ((DistanceSpec(kind="cdtw", window=4), ek.DistanceSpec(kind="cdtw", window=4)),
                          (DistanceSpec(kind="dtw", cost_mode="absolute"),
                           ek.DistanceSpec(kind="dtw", cost_mode="absolute"))):
        for lb in ("none", "keogh", "keogh2"):
            env = refdrive.candidate_envelopes(spec, X, lb)
            for q in Q:
                d, b, cells, comp, ab, skips = refdrive.nn_search(spec, "eapruned", q, X, lb, env)
                rd, rb, st = ek.nn_search(q, X, ek.SearchConfig(spec=refspec, variant="eapruned", lb=lb))
                assert (d, b, cells, comp, ab, skips) == (rd, rb, st.cells, st.computed, st.abandoned, st.lb_skips)
        stream = np.cumsum(rng.normal(size=300))
        for lb in ("none", "keogh2"):
            off, d, cells = refdrive.subsequence_search(spec, "eapruned", Q[0][:30], stream, True, lb=lb)
            ro, rd, st = ek.subsequence_search(Q[0][:30], stream, ek.SearchConfig(spec=refspec, variant="eapruned",
                                                                                   normalize=True, lb=lb))
            assert (off, d, cells) == (ro, rd, st.cells)
