"""All-pairs on equal lengths with the half-warp diagonal engine (E_DIAG4H) stages its series
with compact pads (Params.compact_pad, csrc/ek_kernels.cuh k_triangle): every kind and both
cost modes against the oracle, with the compact layout on and off (EKB_COMPACT_PAD=0)."""

import numpy as np
import pytest

from oracle import eko

pytestmark = pytest.mark.gpu


def _specs(gpu):
    return [gpu.DistanceSpec(kind="cdtw", window=25), gpu.DistanceSpec(kind="erp", erp_gap=0.0, window=25),
            gpu.DistanceSpec(kind="erp", erp_gap=0.3, window=30), gpu.DistanceSpec(kind="msm", msm_c=0.7, window=12),
            gpu.DistanceSpec(kind="twe", twe_nu=0.01, twe_lambda=0.4, window=29),
            gpu.DistanceSpec(kind="wdtw", wdtw_g=0.05, window=20), gpu.DistanceSpec(kind="cdtw", window=0),
            gpu.DistanceSpec(kind="cdtw", window=29, cost_mode="absolute")]


@pytest.mark.parametrize("L", [2, 3, 17, 64, 255, 256, 300])
def test_equal_length_pairwise_compact_pads(gpu, monkeypatch, L):
    rng = np.random.default_rng(1000 + L)
    X = np.cumsum(rng.standard_normal((11, L)), axis=1)
    for spec in _specs(gpu):
        want = eko.pairwise(spec, X, "pruned_only")[0]
        got = gpu.pairwise(spec, X, variant="pruned_only")
        got = got[0] if isinstance(got, tuple) else got
        assert np.array_equal(got, want), (L, spec)
        monkeypatch.setenv("EKB_COMPACT_PAD", "0")
        off = gpu.pairwise(spec, X, variant="pruned_only")
        off = off[0] if isinstance(off, tuple) else off
        monkeypatch.delenv("EKB_COMPACT_PAD")
        assert np.array_equal(off, want), (L, spec)
