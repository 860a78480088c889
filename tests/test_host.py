"""Host-side logic of the drop-in API: validation, orientation, backend seam,
and failing loudly when no GPU is present (there is no CPU fallback)."""

import math
import os

import numpy as np
import pytest

import paper_2102_05221_b200 as ekb
from paper_2102_05221_b200 import DistanceSpec, SearchConfig, SpecError, make_recurrence
from paper_2102_05221_b200._backend import resolve


@pytest.mark.parametrize(
    "kwargs",
    [
        {"kind": "nope"},
        {"kind": "dtw", "cost_mode": "cubed"},
        {"kind": "cdtw"},
        {"kind": "erp", "erp_gap": 0.0},
        {"kind": "erp", "window": 3},
        {"kind": "wdtw"},
        {"kind": "wdtw", "wdtw_g": -0.1},
        {"kind": "msm"},
        {"kind": "msm", "msm_c": -1.0},
        {"kind": "twe"},
        {"kind": "twe", "twe_nu": 0.1},
        {"kind": "twe", "twe_nu": -0.1, "twe_lambda": 1.0},
        {"kind": "dtw", "window": -1},
        {"kind": "dtw", "window": 2.5},
    ],
)
def test_spec_validation_errors(kwargs):
    # the reference's parametrised cases (pkg/tests/test_kernels.py)
    with pytest.raises(SpecError):
        DistanceSpec(**kwargs)


def test_spec_messages_match_reference():
    with pytest.raises(SpecError, match="cdtw requires a finite window"):
        DistanceSpec(kind="cdtw")
    with pytest.raises(SpecError, match="unknown distance kind 'x'"):
        DistanceSpec(kind="x")


def test_effective_window():
    assert DistanceSpec(kind="dtw").effective_window(17) == 17
    assert DistanceSpec(kind="cdtw", window=3).effective_window(17) == 3


def test_orientation_longer_on_rows_ties_keep_first(rng):
    rec = make_recurrence(DistanceSpec(kind="dtw"), rng.normal(0, 1, 4), rng.normal(0, 1, 9))
    assert rec.shape == (9, 4)
    a, b = rng.normal(0, 1, 5), rng.normal(0, 1, 5)
    rec = make_recurrence(DistanceSpec(kind="dtw"), a, b)
    assert rec.lines.tolist() == a.tolist()


def test_as_series_validation():
    with pytest.raises(ValueError):
        ekb.as_series([])
    with pytest.raises(ValueError):
        ekb.as_series([[1.0, 2.0]])
    with pytest.raises(ValueError):
        ekb.as_series([1.0, math.nan])


def test_search_config_validation():
    dtw = DistanceSpec(kind="dtw")
    with pytest.raises(SpecError):
        SearchConfig(spec=dtw, variant="hyper")
    with pytest.raises(SpecError):
        SearchConfig(spec=dtw, lb="keogh3")
    with pytest.raises(SpecError):
        SearchConfig(spec=DistanceSpec(kind="msm", msm_c=0.5), lb="keogh2")
    with pytest.raises(SpecError, match="unknown precision"):
        SearchConfig(spec=dtw, precision="float16")
    assert SearchConfig(spec=dtw, precision="float32").precision == "float32"


def test_spec_struct_matches_header():
    """EkSpec (ctypes) mirrors ek_spec of include/elastik_b200.h, precision last."""
    import re

    from paper_2102_05221_b200 import _lib

    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "include", "elastik_b200.h")).read()
    body = hdr[hdr.index("typedef struct ek_spec {"):hdr.index("} ek_spec;")]
    names = re.findall(r"\b(\w+);", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert names == [f[0] for f in _lib.EkSpec._fields_]
    with pytest.raises(SpecError, match="unknown precision"):
        _lib.SpecHandle(DistanceSpec(kind="dtw"), precision="half")


def test_backend_seam():
    with pytest.raises(ValueError):
        resolve("turbo")
    with pytest.raises(RuntimeError):
        resolve("python")  # the reference's CPU engines are not part of this build


def test_no_silent_cpu_fallback():
    if ekb.compiled_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        ekb.distance(DistanceSpec(kind="dtw"), "base", [1.0, 2.0], [1.0])
    with pytest.raises(RuntimeError):
        ekb.nn_search([1.0, 2.0], [[1.0]], SearchConfig(spec=DistanceSpec(kind="dtw")))


def test_facade_rejects_unknown_variant():
    with pytest.raises(SpecError):
        ekb.distance(DistanceSpec(kind="dtw"), "fast", [1.0], [2.0])


def test_wdtw_table_is_libm(rng):
    t = ekb.wdtw_weight_table(0.17, 219)
    for d in rng.integers(0, 220, size=5):
        assert t[int(d)] == 1.0 / (1.0 + math.exp(-0.17 * (int(d) - 219 / 2.0)))


def test_generator_is_seeded():
    from paper_2102_05221_b200 import datagen

    a = datagen.warped_prototypes(5, 64, 2, 0.1, 3)
    b = datagen.warped_prototypes(5, 64, 2, 0.1, 3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.allclose(a[0].mean(axis=1), 0, atol=1e-12)


# ---- the Recurrence payload (kernels.py:128-154, 264-277): the reference's own kernel tests
# (pkg/tests/test_kernels.py:119-162) restated, plus a check of every closure against the
# live reference's where it is importable (this container)

def test_erp_border_prefix():
    rec = make_recurrence(DistanceSpec(kind="erp", window=2, erp_gap=0.0), [3.0, 1.0], [3.0, 1.0])
    assert rec.init_v_border(1) == 9.0
    assert rec.init_v_border(2) == 10.0
    assert rec.init_corner == 0.0
    assert rec.v_border_vals.tolist() == [0.0, 9.0, 10.0]


def test_msm_canonical_is_absolute_regardless_of_mode():
    for mode in ("squared", "absolute"):
        rec = make_recurrence(DistanceSpec(kind="msm", msm_c=0.5, cost_mode=mode), [4.0, 0.0], [1.0, 0.0])
        assert rec.canonical(1, 1) == 3.0


def test_dtw_borders_are_infinite():
    rec = make_recurrence(DistanceSpec(kind="dtw"), [1.0, 2.0], [3.0, 4.0])
    for k in (1, 2):
        assert math.isinf(rec.init_h_border(k))
        assert math.isinf(rec.init_v_border(k))
    assert rec.v_border_vals is None and rec.h_border_vals is None


def _specs(rng, maxlen, mode="squared"):
    return [DistanceSpec(kind="dtw", cost_mode=mode), DistanceSpec(kind="cdtw", window=3, cost_mode=mode),
            DistanceSpec(kind="wdtw", wdtw_g=float(rng.uniform(0, 0.5)), cost_mode=mode),
            DistanceSpec(kind="erp", window=int(rng.integers(0, maxlen)), erp_gap=float(rng.uniform(-1, 1)),
                         cost_mode=mode),
            DistanceSpec(kind="msm", msm_c=float(rng.uniform(0, 2)), cost_mode=mode),
            DistanceSpec(kind="twe", twe_nu=float(rng.uniform(0, 1)), twe_lambda=float(rng.uniform(0, 2)),
                         cost_mode=mode)]


def test_border_monotonicity_and_nonnegative_moves(rng):
    for mode in ("squared", "absolute"):
        for spec in _specs(rng, 10, mode):
            rec = make_recurrence(spec, rng.uniform(-9, 9, 10), rng.uniform(-9, 9, 8))
            nl, nc = rec.shape
            vb = [rec.init_v_border(i) for i in range(1, nl + 1)]
            hb = [rec.init_h_border(j) for j in range(1, nc + 1)]
            assert all(a <= b for a, b in zip(vb, vb[1:]))
            assert all(a <= b for a, b in zip(hb, hb[1:]))
            for i in range(1, nl + 1):
                for j in range(1, nc + 1):
                    assert rec.canonical(i, j) >= 0.0 and rec.alt_row(i, j) >= 0.0 and rec.alt_col(i, j) >= 0.0


def test_recurrence_closures_equal_the_live_reference(rng):
    """Every closure value and payload array bit-equal to the reference's make_recurrence."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import refpkg

    ek = refpkg.load()
    if ek is None:
        pytest.skip("reference package not present (GPU box)")
    for mode in ("squared", "absolute"):
        for spec in _specs(rng, 12, mode):
            refspec = ek.DistanceSpec(**{k: getattr(spec, k) for k in ("kind", "window", "wdtw_g", "erp_gap", "msm_c",
                                                                        "twe_nu", "twe_lambda", "cost_mode")})
            for orient in ("auto", "st"):
                a, b = rng.normal(0, 2, int(rng.integers(1, 12))), rng.normal(0, 2, int(rng.integers(1, 12)))
                ours, ref = make_recurrence(spec, a, b, orient), ek.kernels.make_recurrence(refspec, a, b, orient)
                assert ours.shape == ref.shape
                nl, nc = ours.shape
                for name in ("canonical", "alt_row", "alt_col"):
                    f, g = getattr(ours, name), getattr(ref, name)
                    assert [f(i, j) for i in range(1, nl + 1) for j in range(1, nc + 1)] == \
                        [g(i, j) for i in range(1, nl + 1) for j in range(1, nc + 1)], (spec.kind, name)
                assert [ours.init_v_border(i) for i in range(1, nl + 1)] == [ref.init_v_border(i) for i in range(1, nl + 1)]
                assert [ours.init_h_border(j) for j in range(1, nc + 1)] == [ref.init_h_border(j) for j in range(1, nc + 1)]
                for name in ("wdtw_weights", "v_border_vals", "h_border_vals"):
                    x, y = getattr(ours, name), getattr(ref, name)
                    assert (x is None) == (y is None) and (x is None or np.array_equal(x, y)), name
