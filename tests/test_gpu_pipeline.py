"""The streaming 1-NN entry (search.NNPipeline / nn_batch_stream over ek_nn_submit /
ek_nn_collect): every batch's answers equal nn_batch's and the oracle's, whatever the
batches in flight around it (sizes, kinds, lengths), and errors surface at the batch that
caused them without disturbing the other slot."""

import numpy as np
import pytest

from oracle import eko

pytestmark = pytest.mark.gpu


def _batches(gpu, rng):
    from paper_2102_05221_b200 import datagen

    out = []
    Q, _, C, _ = datagen.C2.make(n_queries=24, n_candidates=600)
    out.append((gpu.DistanceSpec(kind="cdtw", window=51), Q, C))
    out.append((gpu.DistanceSpec(kind="dtw"), rng.normal(size=(5, 64)).cumsum(1), rng.normal(size=(70, 64)).cumsum(1)))
    out.append((gpu.DistanceSpec(kind="msm", msm_c=0.5), rng.normal(size=(3, 50)).cumsum(1),
                [rng.normal(size=int(n)).cumsum() for n in rng.integers(30, 70, 40)]))
    out.append((gpu.DistanceSpec(kind="cdtw", window=51), Q[:7], C[::3].copy()))
    return out


def test_pipeline_matches_nn_batch_and_oracle(gpu, rng):
    batches = _batches(gpu, rng)
    want = [gpu.nn_batch(s, "eapruned", q, c) for s, q, c in batches]
    for spec, q, c in batches[1:3]:  # small ones against the oracle too
        ref = eko.nn(spec, "eapruned", q, c)
        got = gpu.nn_batch(spec, "eapruned", q, c)
        assert np.array_equal(got[0], ref["nn_index"]) and np.array_equal(got[1], ref["nn_distance"])
    # one spec per pipeline: run each spec's batches as a stream, interleaving sizes
    for spec_i in range(len(batches)):
        spec = batches[spec_i][0]
        same = [(q, c) for s, q, c in batches if s == spec] * 3
        exp = [w for (s, _, _), w in zip(batches, want) if s == spec] * 3
        got = list(gpu.nn_batch_stream(spec, "eapruned", same))
        assert len(got) == len(exp)
        for g, w in zip(got, exp):
            assert np.array_equal(g[0], w[0]) and np.array_equal(g[1], w[1])


def test_pipeline_manual_submit_collect(gpu, rng):
    spec = gpu.DistanceSpec(kind="cdtw", window=6)
    Q1, C1 = rng.normal(size=(9, 60)).cumsum(1), rng.normal(size=(200, 60)).cumsum(1)
    Q2, C2 = rng.normal(size=(4, 60)).cumsum(1), rng.normal(size=(100, 60)).cumsum(1)
    pipe = gpu.NNPipeline(spec, "eapruned")
    pipe.submit(Q1, C1)
    pipe.submit(Q2, C2)
    with pytest.raises(gpu.SearchError):
        pipe.submit(Q1, C1)  # two in flight
    a = pipe.collect()
    b = pipe.collect()
    for got, (q, c) in ((a, (Q1, C1)), (b, (Q2, C2))):
        ref = eko.nn(spec, "eapruned", q, c)
        assert np.array_equal(got[0], ref["nn_index"]) and np.array_equal(got[1], ref["nn_distance"])
    with pytest.raises(gpu.SearchError):
        pipe.collect()


def test_pipeline_nonfinite_batch_raises_and_other_slot_survives(gpu, rng):
    spec = gpu.DistanceSpec(kind="cdtw", window=4)
    Q, C = rng.normal(size=(3, 40)), rng.normal(size=(50, 40))
    Cb = C.copy()
    Cb[7, 3] = np.nan
    pipe = gpu.NNPipeline(spec, "eapruned")
    pipe.submit(Q, C)
    pipe.submit(Q, Cb)
    good = pipe.collect()
    with pytest.raises(ValueError, match="must all be finite"):
        pipe.collect()
    ref = eko.nn(spec, "eapruned", Q, C)
    assert np.array_equal(good[0], ref["nn_index"]) and np.array_equal(good[1], ref["nn_distance"])
    # the library and the pipeline stay usable
    pipe.submit(Q, C)
    again = pipe.collect()
    assert np.array_equal(again[0], good[0]) and np.array_equal(again[1], good[1])
