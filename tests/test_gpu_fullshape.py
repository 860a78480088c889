"""Parity at the EXACT BASELINE.json shapes (bench.py's inputs, rank 0's seeds) against the
C oracle (oracle/ek_oracle.c, pinned to the live reference in tests/test_oracle_pins.py),
run with every host thread:

* C1: DTW 1-NN, all 16 queries x 256 candidates, L=128;
* C2: CDTW(w=51) 1-NN, all 256 queries x 4096 candidates, L=512;
* C3: the full 1024 x 1024 pruned_only matrices for WDTW(g=0.05) and ERP(gap 0, w=25);
* C4: MSM(c=1) and TWE(nu=0.001, lambda=1) 1-NN, 64 of 512 queries x 8192 candidates;
* C5: CDTW(w=51) z-normalised subsequence search, query 1024 on the 2^20-point stream.

Bit-exact: nn indices and distances, every matrix entry, the best (offset, distance).
"""

import os

import numpy as np
import pytest

from oracle import eko

pytestmark = pytest.mark.gpu

THREADS = len(os.sched_getaffinity(0))


def _bench():
    import bench

    return bench


@pytest.mark.parametrize("name,nq", [("c1", None), ("c2", None), ("c4m", 64), ("c4t", 64)])
def test_nn_exact_shape(gpu, name, nq):
    b = _bench()
    wl, Q, ql, C, cl = b.nn_data(name, 0)
    assert (Q.shape, C.shape) == ((wl.n_queries, wl.length), (wl.n_candidates, wl.length))
    spec = b.spec_for(name)
    idx, dist = gpu.nn_batch(spec, "eapruned", Q, C)[:2]
    Qs = Q if nq is None else Q[:: Q.shape[0] // nq][:nq]
    want = eko.nn(spec, "eapruned", Qs, C, threads=THREADS)
    sel = slice(None) if nq is None else slice(None, None, Q.shape[0] // nq)
    got_i, got_d = idx[sel][: len(Qs)], dist[sel][: len(Qs)]
    assert np.array_equal(got_i, want["nn_index"]), np.nonzero(got_i != want["nn_index"])
    assert np.array_equal(got_d.view(np.int64), want["nn_distance"].view(np.int64))
    # labels follow (classify_1nn)
    assert np.array_equal(cl[got_i], cl[want["nn_index"]])


@pytest.mark.parametrize("name", ["c3w", "c3e"])
def test_pairwise_exact_shape(gpu, name):
    b = _bench()
    from paper_2102_05221_b200 import datagen

    X, _ = datagen.pairwise_workload()
    assert X.shape == (1024, 256)
    spec = b.spec_for(name)
    D, _ = gpu.pairwise(spec, X, variant="pruned_only")
    Dw, _ = eko.pairwise(spec, X, threads=THREADS)
    assert np.array_equal(D.view(np.int64), Dw.view(np.int64)), int(np.sum(D != Dw))
    assert np.array_equal(D, D.T) and not np.diag(D).any()


def test_subsequence_exact_shape(gpu):
    b = _bench()
    from paper_2102_05221_b200 import datagen

    stream, q = datagen.subsequence_workload()
    assert (len(stream), len(q)) == (1 << 20, 1024)
    spec = b.spec_for("c5")
    got = gpu.subsequence_search(q, stream, gpu.SearchConfig(spec=spec, variant="eapruned", normalize=True))[:2]
    want = eko.subsequence(spec, "eapruned", q, stream, True, chunk=8192, threads=THREADS)[:2]
    assert got[0] == want[0] and np.float64(got[1]).view(np.int64) == np.float64(want[1]).view(np.int64), (got, want)
