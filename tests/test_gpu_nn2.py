"""k_nn2 (csrc/ek_nn2.cuh): the LB path's two-pairs-per-warp phase B with per-query work
counters.  Shapes cover one query, query counts that are not multiples of 8 or that span
several 64-bit words of the done bitmask, bands with and without both virtual diagonals in
slot 0 (VIRT0), unconstrained dtw on short series, both cost modes, the FP32 mode, planted
duplicates (lowest index wins) and the ea / eapruned variants.  Each run is compared with
the oracle's serial scan, and with the one-pair-per-warp kernel (EKB_NN2=0).
"""

import numpy as np
import pytest

from oracle import eko

pytestmark = pytest.mark.gpu


def _data(rng, nq, nc, L):
    from paper_2102_05221_b200 import datagen

    C, _, protos = datagen.warped_prototypes(nc, L, 8, 0.1, int(rng.integers(1 << 30)))
    Q, _, _ = datagen.warped_prototypes(nq, L, 8, 0.1, int(rng.integers(1 << 30)), protos=protos)
    if nq > 2:
        Q[1] = C[nc // 3]  # distance 0, duplicated at a higher index: the lower one wins
        C[nc // 3 + 5] = C[nc // 3]
    return Q, C


@pytest.mark.parametrize(
    "nq,nc,L,kind,window,mode",
    [
        (1, 300, 64, "cdtw", 6, "squared"),      # band not VIRT0 (w even)
        (7, 500, 96, "cdtw", 11, "absolute"),    # VIRT0
        (65, 400, 64, "cdtw", 10, "squared"),    # two bitmask words
        (130, 257, 48, "cdtw", 5, "squared"),    # three words, odd candidate count
        (33, 600, 200, "cdtw", 51, "squared"),   # the C2 band on shorter series
        (20, 300, 40, "dtw", None, "squared"),   # unconstrained, 2L - 1 diagonals <= 128 slots
    ],
)
def test_nn2_matches_oracle_and_one_pair_kernel(gpu, rng, monkeypatch, nq, nc, L, kind, window, mode):
    Q, C = _data(rng, nq, nc, L)
    spec = gpu.DistanceSpec(kind=kind, window=window, cost_mode=mode)
    for variant in ("eapruned", "ea"):
        r = eko.nn(spec, variant, Q, C, threads=8)
        for nn2 in ("1", "0"):
            monkeypatch.setenv("EKB_NN2", nn2)
            idx, dist, cells, comp, ab = gpu.nn_batch(spec, variant, Q, C)
            assert np.array_equal(idx, r["nn_index"]), (variant, nn2)
            assert np.array_equal(dist, r["nn_distance"]), (variant, nn2)
            assert np.all(comp + ab == nc)
        if nq > 2:
            assert idx[1] == nc // 3 and dist[1] == 0.0


def test_nn2_fp32_mode(gpu, rng, monkeypatch):
    Q, C = _data(rng, 40, 700, 128)
    spec = gpu.DistanceSpec(kind="cdtw", window=13)
    r = eko.nn(spec, "eapruned", Q, C, threads=8)
    monkeypatch.setenv("EKB_NN2", "1")
    idx, dist = gpu.nn_batch(spec, "eapruned", Q, C, precision="float32")[:2]
    rel = np.abs(dist - r["nn_distance"]) / np.maximum(r["nn_distance"], 1e-300)
    assert np.all(rel <= 1e-5)
    # index mismatches only on near ties (as tests/test_gpu_fp32.py)
    for q in np.flatnonzero(idx != r["nn_index"]):
        d_alt = eko.distance(spec, "base", Q[q], C[idx[q]])[0]
        assert abs(d_alt - r["nn_distance"][q]) <= 1e-5 * r["nn_distance"][q]
