"""Ingestion on the device: resident batches, series.derivative and
series.znormalize on the GPU bit-for-bit against the reference's numpy formulas
(pkg/src/elastik/series.py:118-144; pinned by pkg/tests/test_series.py:104-156), and
1-NN on resident batches equal to the host-array path and the oracle."""

import numpy as np
import pytest

from oracle import eko

pytestmark = pytest.mark.gpu


def _ragged(rng, n, lo, hi):
    out = [np.cumsum(rng.normal(size=int(rng.integers(lo, hi)))) for _ in range(n)]
    out[0] = np.full(len(out[0]), 3.25)          # constant: znormalize -> zeros
    out[1] = np.array([1.0, 2.0, 4.0])           # the shortest legal derivative input
    out[2] = rng.normal(size=1000) * 1e-13       # std below 1e-12 -> zeros
    out[3] = np.array([5.0, -5.0])               # two points
    return out


def test_upload_round_trip_and_pinned_load(gpu, rng, tmp_path):
    from paper_2102_05221_b200 import ingest, series

    xs = _ragged(rng, 40, 2, 700)
    with ingest.DeviceSeries.upload(xs) as d:
        back = d.to_host()
    assert all(a.tobytes() == b.tobytes() for a, b in zip(xs, back))
    p = tmp_path / "x.tsv"
    series.write_tsv(series.LabeledDataset("x", tuple((k % 3, x) for k, x in enumerate(xs))), p)
    pk = ingest.load_tsv_packed(p)
    assert pk.pinned  # page-locked when a device is present
    with ingest.DeviceSeries.upload(pk) as d:
        assert all(a.tobytes() == b.tobytes() for a, b in zip(xs, d.to_host()))


def test_derivative_and_znormalize_bit_exact(gpu, rng):
    from paper_2102_05221_b200 import ingest, series

    xs = _ragged(rng, 300, 3, 3000)
    xs.append(rng.normal(size=200_000).cumsum())   # long series: deep pairwise-sum recursion
    x3 = [x for x in xs if len(x) >= 3]
    with ingest.DeviceSeries.upload(x3) as d:
        with d.derivative() as dd:
            got = dd.to_host()
        want = [series.derivative(x) for x in x3]
        assert all(a.tobytes() == b.tobytes() for a, b in zip(got, want))
    with ingest.DeviceSeries.upload(xs) as d:
        with d.znormalize() as dz:
            got = dz.to_host()
        want = [series.znormalize(x) for x in xs]
        assert all(a.tobytes() == b.tobytes() for a, b in zip(got, want))
        # the reference's formulas directly (np.mean / np.std, the derivative expression)
        x = xs[10]
        assert got[10].tobytes() == ((x - x.mean()) / x.std()).tobytes()


def test_transform_length_errors(gpu):
    from paper_2102_05221_b200 import ingest
    from paper_2102_05221_b200.errors import DegenerateInputError

    with ingest.DeviceSeries.upload([np.array([1.0, 2.0]), np.array([1.0, 2.0, 3.0])]) as d:
        with pytest.raises(DegenerateInputError):
            d.derivative()
    with ingest.DeviceSeries.upload([np.array([1.0])]) as d:
        with pytest.raises(DegenerateInputError):
            d.znormalize()
    with pytest.raises(ValueError):
        ingest.DeviceSeries.upload([np.array([1.0, np.nan])])


@pytest.mark.parametrize("kind,window", [("cdtw", 9), ("msm", None), ("dtw", None)])
def test_nn_on_resident_batches(gpu, rng, kind, window):
    from paper_2102_05221_b200 import datagen, ingest

    C, _, protos = datagen.warped_prototypes(500, 96, 6, 0.1, 5)
    Q, _, _ = datagen.warped_prototypes(24, 96, 6, 0.1, 6, protos=protos)
    params = {"msm": dict(msm_c=1.0)}.get(kind, {})
    spec = gpu.DistanceSpec(kind=kind, window=window, **params)
    want = eko.nn(spec, "eapruned", Q, C, threads=8)
    with ingest.DeviceSeries.upload(Q) as dq, ingest.DeviceSeries.upload(C) as dc:
        idx, dist, cells, comp, ab = ingest.nn_batch_device(spec, "eapruned", dq, dc)
        # a derived batch (two points shorter) stays on the device for the next search
        with dq.derivative() as dq2, dc.derivative() as dc2:
            i2, d2 = ingest.nn_batch_device(spec, "eapruned", dq2, dc2)[:2]
    assert np.array_equal(idx, want["nn_index"]) and np.array_equal(dist, want["nn_distance"])
    from paper_2102_05221_b200 import series
    Qd = np.stack([series.derivative(q) for q in Q])
    Cd = np.stack([series.derivative(c) for c in C])
    w2 = eko.nn(spec, "eapruned", Qd, Cd, threads=8)
    assert np.array_equal(i2, w2["nn_index"]) and np.array_equal(d2, w2["nn_distance"])
    h = gpu.nn_batch(spec, "eapruned", Q, C)
    assert np.array_equal(h[0], idx) and np.array_equal(h[1], dist)


def test_nn_on_ragged_resident_batches(gpu, rng):
    from paper_2102_05221_b200 import ingest

    C = [np.cumsum(rng.normal(size=int(rng.integers(20, 90)))) for _ in range(200)]
    Q = [np.cumsum(rng.normal(size=int(rng.integers(20, 90)))) for _ in range(10)]
    spec = gpu.DistanceSpec(kind="cdtw", window=30)
    want = eko.nn(spec, "eapruned", Q, C, threads=8)
    with ingest.DeviceSeries.upload(Q) as dq, ingest.DeviceSeries.upload(C) as dc:
        idx, dist = ingest.nn_batch_device(spec, "eapruned", dq, dc)[:2]
    assert np.array_equal(idx, want["nn_index"]) and np.array_equal(dist, want["nn_distance"])
