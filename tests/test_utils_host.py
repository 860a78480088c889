"""Host utilities of the drop-in API against fixtures from the live reference
(tests/golden/make_golden_utils.py) and the reference's own known answers
(pkg/tests/test_lower_bounds.py, test_series.py).  CPU only."""

import os

import numpy as np
import pytest

import paper_2102_05221_b200 as ekb
from paper_2102_05221_b200 import ParseError

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "utils.npz"))


def test_envelope_and_lb_match_reference():
    off = 0
    for k, n in enumerate(G["lens"]):
        s, t = G["S"][off:off + n], G["T"][off:off + n]
        w = int(G["wins"][k])
        mode = "squared" if G["modes"][k] else "absolute"
        env = ekb.build_envelope(s, w)
        assert np.array_equal(env.upper, G["upper"][off:off + n])
        assert np.array_equal(env.lower, G["lower"][off:off + n])
        assert ekb.lb_keogh(t, env, mode) == G["lb"][k]
        off += n


def test_lb_keogh2_matches_reference():
    off = 0
    for k, n in enumerate(G["lens"]):
        s, t = G["S"][off:off + n], G["T"][off:off + n]
        w = int(G["wins"][k])
        mode = "squared" if G["modes"][k] else "absolute"
        es, et = ekb.build_envelope(s, w), ekb.build_envelope(t, w)
        assert ekb.lb_keogh2(t, s, es, et, cutoff=float(G["lb2_cut"][k]), cost_mode=mode) == G["lb2"][k]
        off += n


def test_known_answers():
    env = ekb.build_envelope([1.0, 3.0, 2.0], 1)
    assert env.upper.tolist() == [3.0, 3.0, 3.0] and env.lower.tolist() == [1.0, 1.0, 2.0]
    assert ekb.lb_keogh([0.0, 0.0, 0.0], env, "squared") == 6.0
    s = np.arange(5.0)
    assert ekb.build_envelope(s, 0).upper.tolist() == s.tolist()
    with pytest.raises(ekb.DimensionError):
        ekb.lb_keogh([1.0, 2.0, 3.0], ekb.build_envelope([1.0, 2.0], 1))
    with pytest.raises(ValueError):
        ekb.build_envelope([1.0], -1)


def test_envelope_naive(rng):
    for _ in range(200):
        n = int(rng.integers(1, 60))
        w = int(rng.integers(0, n + 3))
        s = rng.normal(0, 2, n)
        env = ekb.build_envelope(s, w)
        assert env.upper.tolist() == [max(s[max(0, i - w): i + w + 1]) for i in range(n)]
        assert env.lower.tolist() == [min(s[max(0, i - w): i + w + 1]) for i in range(n)]


def test_lb_keogh_below_gpu_free_oracle(rng):
    from oracle import eko

    for _ in range(100):
        n = int(rng.integers(2, 40))
        w = int(rng.integers(0, n))
        mode = "squared" if rng.random() < 0.5 else "absolute"
        q, c = np.cumsum(rng.normal(0, 1, n)), np.cumsum(rng.normal(0, 1, n))
        spec = ekb.DistanceSpec(kind="cdtw", window=w, cost_mode=mode)
        exact = eko.distance(spec, "base", q, c)[0]
        assert ekb.lb_keogh(q, ekb.build_envelope(c, w), mode) <= exact


def test_derivative_and_random_walk():
    assert np.array_equal(ekb.derivative(G["deriv_in"]), G["deriv_out"])
    with pytest.raises(ekb.DegenerateInputError):
        ekb.derivative([1.0, 2.0])
    ds = ekb.gen_random_walk(9, 31, 4, seed=12)
    assert ds.labels == G["rw_labels"].tolist()
    assert np.array_equal(np.stack(ds.series), G["rw_series"])


def test_tsv_roundtrip_and_errors(tmp_path):
    ds = ekb.gen_random_walk(9, 31, 4, seed=12)
    p = tmp_path / "x.tsv"
    ekb.write_tsv(ds, p, delimiter="comma")
    assert p.read_text(encoding="utf-8") == str(G["tsv_text"])
    back = ekb.load_tsv(p, delimiter="comma")
    assert back.labels == ds.labels
    assert all(np.array_equal(a, b) for a, b in zip(back.series, ds.series))
    q = tmp_path / "y.tsv"
    q.write_bytes(b"1\t0.5\t1.5\r\n\r\n2.9\t3\t4\r\n")
    y = ekb.load_tsv(q)
    assert y.labels == [1, 2] and y.series[1].tolist() == [3.0, 4.0]
    bad = tmp_path / "bad.tsv"
    bad.write_text("1\t0.5\n2\tx\t1\n")
    with pytest.raises(ParseError, match="line 2, column 2"):
        ekb.load_tsv(bad)
    bad.write_text("1\t0.5\n2\tnan\n")
    with pytest.raises(ParseError, match="non-finite"):
        ekb.load_tsv(bad)
    bad.write_text("\n\n")
    with pytest.raises(ekb.EmptyDatasetError):
        ekb.load_tsv(bad)
    with pytest.raises(ValueError):
        ekb.load_tsv(p, delimiter="space")
