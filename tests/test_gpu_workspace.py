"""The per-stream workspace of the 1-NN and subsequence entries (csrc/ek_api.cu: ArenaScope):
calls of growing and shrinking sizes on one stream, kinds that take different scratch
layouts back to back, the resident entry on two torch streams, and EKB_WORKSPACE=0 (plain
stream-ordered allocations) must all return the answers of the oracle's serial scan.
"""

import numpy as np
import pytest

from oracle import eko

pytestmark = pytest.mark.gpu


def _data(seed, nq, nc, L):
    from paper_2102_05221_b200 import datagen

    C, _, protos = datagen.warped_prototypes(nc, L, 6, 0.1, seed)
    Q, _, _ = datagen.warped_prototypes(nq, L, 6, 0.1, seed + 1, protos=protos)
    return Q, C


def _check(ekb, spec, Q, C):
    idx, dist, *_ = ekb.nn_batch(spec, "eapruned", Q, C)
    ref = eko.nn(spec, "eapruned", Q, C)
    assert np.array_equal(idx, ref["nn_index"])
    assert np.array_equal(dist, ref["nn_distance"])


def test_workspace_grows_shrinks_and_changes_layout(gpu, monkeypatch):
    import paper_2102_05221_b200 as ekb

    cdtw = ekb.DistanceSpec(kind="cdtw", window=9)
    msm = ekb.DistanceSpec(kind="msm", msm_c=0.5)
    twe = ekb.DistanceSpec(kind="twe", twe_nu=0.01, twe_lambda=0.5)
    shapes = [(3, 40, 64), (40, 900, 96), (5, 33, 48), (64, 1500, 80), (2, 10, 32)]
    for rep in range(2):
        for k, (nq, nc, L) in enumerate(shapes):
            Q, C = _data(100 * rep + k, nq, nc, L)
            _check(ekb, cdtw, Q, C)  # LB path: envelopes, keys, ranks, padded copies
            if nc <= 900:
                _check(ekb, msm if k % 2 else twe, Q[: min(nq, 6)], C)  # ranked path: PAA keys, overflow lists
    monkeypatch.setenv("EKB_WORKSPACE", "0")
    Q, C = _data(7, 17, 300, 72)
    _check(ekb, cdtw, Q, C)
    monkeypatch.delenv("EKB_WORKSPACE")
    _check(ekb, cdtw, Q, C)


def test_workspace_per_stream_resident_entry(gpu):
    import torch

    import paper_2102_05221_b200 as ekb
    from paper_2102_05221_b200 import _lib

    L = _lib.lib()
    spec = ekb.DistanceSpec(kind="cdtw", window=7)
    h = _lib.SpecHandle(spec, longest_lengths=[64])
    dev = torch.device("cuda", 0)
    jobs = []
    for s_i, (nq, nc) in enumerate([(24, 700), (9, 1300)]):
        Q, C = _data(50 + s_i, nq, nc, 64)
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
        jobs.append(dict(Q=Q, C=C, dQ=t(Q.reshape(-1), torch.float64), dC=t(C.reshape(-1), torch.float64),
                         qo=t(np.arange(nq) * 64, torch.int64), co=t(np.arange(nc) * 64, torch.int64),
                         ql=t(np.full(nq, 64), torch.int32), cl=t(np.full(nc, 64), torch.int32),
                         out=torch.empty(5 * nq, dtype=torch.int64, device=dev), st=torch.cuda.Stream(device=dev)))
    torch.cuda.synchronize()
    for rep in range(3):  # interleaved calls on two streams: each keeps its own workspace
        for j in jobs:
            nq, nc = j["Q"].shape[0], j["C"].shape[0]
            o = j["out"].data_ptr()
            _lib.check(L.ek_nn_dev(h.ref, 2, j["dQ"].data_ptr(), j["qo"].data_ptr(), j["ql"].data_ptr(), nq,
                                   j["dC"].data_ptr(), j["co"].data_ptr(), j["cl"].data_ptr(), nc, 64, 1, o,
                                   o + 8 * nq, o + 16 * nq, o + 24 * nq, o + 32 * nq, j["st"].cuda_stream))
    torch.cuda.synchronize()
    for j in jobs:
        nq = j["Q"].shape[0]
        ref = eko.nn(spec, "eapruned", j["Q"], j["C"])
        out = j["out"].cpu().numpy()
        assert np.array_equal(out[:nq], ref["nn_index"])
        assert np.array_equal(out[nq: 2 * nq].view(np.float64), ref["nn_distance"])


def test_workspace_subsequence_repeat(gpu):
    import paper_2102_05221_b200 as ekb
    from paper_2102_05221_b200 import SearchConfig

    rng = np.random.default_rng(11)
    for n, lq in ((3000, 64), (20000, 128), (1500, 32)):
        stream = np.cumsum(rng.standard_normal(n))
        q = np.cumsum(rng.standard_normal(lq))
        spec = ekb.DistanceSpec(kind="cdtw", window=max(1, lq // 20))
        got = ekb.subsequence_search(q, stream, SearchConfig(spec=spec, variant="eapruned", normalize=True))[:2]
        want = eko.subsequence(spec, "eapruned", q, stream, True, chunk=512, threads=4)[:2]
        assert got == want, (n, lq)


def test_subsequence_plan_cache_eviction(gpu):
    """More query lengths than the per-length plan cache keeps (64): the cache is dropped and
    rebuilt, and the answers stay the oracle's."""
    import paper_2102_05221_b200 as ekb
    from paper_2102_05221_b200 import SearchConfig

    rng = np.random.default_rng(23)
    stream = np.cumsum(rng.standard_normal(1200))
    for lq in list(range(8, 80)) + [8, 40, 79]:
        q = np.cumsum(rng.standard_normal(lq))
        spec = ekb.DistanceSpec(kind="cdtw", window=max(1, lq // 10))
        got = ekb.subsequence_search(q, stream, SearchConfig(spec=spec, variant="eapruned", normalize=True))[:2]
        if lq % 9 == 0 or lq in (8, 79):
            want = eko.subsequence(spec, "eapruned", q, stream, True, chunk=512, threads=4)[:2]
            assert got == want, lq
