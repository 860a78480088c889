"""Seeded synthetic workloads for the BASELINE.json configs.

The reference has no such generator (its ``gen_random_walk``,
pkg/src/elastik/series.py:147-170, only drifts random walks per class) and
the paper's UCR archive is not available, so these inputs stand in for it
with the shapes, sizes and value distributions BASELINE.json names:

* class prototype  = cumsum of N(0,1) increments, length L;
* warp             = monotone piecewise-linear map output index -> source
                     position, endpoints 0 and L-1, 5 interior knots at
                     k(L-1)/6 offset by U(-0.1L, +0.1L), sorted and clipped;
* sample           = prototype linearly interpolated at the warped positions
                     + N(0, sigma) noise, then z-normalised (numpy mean/std,
                     the arithmetic of series.znormalize, series.py:118-131);
* labels           = uniform over the classes.

Every choice lives here and is echoed into bench results (``describe``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _znorm_rows(x: np.ndarray) -> np.ndarray:
    out = np.empty_like(x)
    for k in range(x.shape[0]):
        s = x[k]
        mean = s.mean()
        std = s.std()
        out[k] = 0.0 if std < 1e-12 else (s - mean) / std
    return out


def warped_prototypes(n: int, length: int, classes: int, sigma: float, seed: int,
                      protos: np.ndarray | None = None):
    """Return (X[n, L] float64 z-normalised, labels[n] int64, prototypes[classes, L])."""
    rng = np.random.default_rng(seed)
    if protos is None:
        protos = np.cumsum(rng.normal(0.0, 1.0, size=(classes, length)), axis=1)
    labels = rng.integers(0, classes, size=n).astype(np.int64)
    grid = np.arange(length, dtype=np.float64)
    knots_x = np.linspace(0.0, length - 1.0, 7)
    X = np.empty((n, length), dtype=np.float64)
    for k in range(n):
        off = rng.uniform(-0.1 * length, 0.1 * length, size=5)
        knots_y = knots_x.copy()
        knots_y[1:6] = np.clip(np.sort(knots_x[1:6] + off), 0.0, length - 1.0)
        pos = np.interp(grid, knots_x, knots_y)
        X[k] = np.interp(pos, grid, protos[labels[k]]) + rng.normal(0.0, sigma, size=length)
    return _znorm_rows(X), labels, protos


@dataclass(frozen=True)
class NNWorkload:
    name: str
    kind: str
    n_queries: int
    n_candidates: int
    length: int
    classes: int
    sigma: float
    seed: int

    def make(self, n_queries: int | None = None, n_candidates: int | None = None):
        """(Q, q_labels, C, c_labels); train and test share the class prototypes."""
        nq = self.n_queries if n_queries is None else n_queries
        nc = self.n_candidates if n_candidates is None else n_candidates
        C, cl, protos = warped_prototypes(self.n_candidates, self.length, self.classes, self.sigma,
                                          self.seed)
        Q, ql, _ = warped_prototypes(self.n_queries, self.length, self.classes, self.sigma,
                                     self.seed + 1, protos=protos)
        return Q[:nq], ql[:nq], C[:nc], cl[:nc]


# BASELINE.json configs[0], [1], [3]
C1 = NNWorkload("c1_dtw_nn", "dtw", 16, 256, 128, 8, 0.1, 1001)
C2 = NNWorkload("c2_cdtw_nn", "cdtw", 256, 4096, 512, 16, 0.1, 2002)
C4 = NNWorkload("c4_msm_twe_nn", "msm", 512, 8192, 512, 32, 0.2, 4004)


def pairwise_workload(n: int = 1024, length: int = 256, classes: int = 8, seed: int = 3003):
    """BASELINE.json configs[2]: 1024 series of length 256, 8 classes."""
    X, labels, _ = warped_prototypes(n, length, classes, 0.1, seed)
    return X, labels


def subsequence_workload(stream_len: int = 1 << 20, query_len: int = 1024, seed: int = 5005):
    """BASELINE.json configs[4]: a 2^20-point N(0,1)-increment random walk stream and an
    independent z-normalised random-walk query of length 1024."""
    rng = np.random.default_rng(seed)
    stream = np.cumsum(rng.normal(0.0, 1.0, size=stream_len))
    q = np.cumsum(rng.normal(0.0, 1.0, size=query_len))
    return stream, _znorm_rows(q[None, :])[0]


def describe():
    return {
        "generator": "warped-prototype (paper_2102_05221_b200/datagen.py)",
        "prototype": "cumsum N(0,1)",
        "warp": "piecewise-linear, 5 interior knots, offsets U(-0.1L,0.1L)",
        "znorm": "per series (numpy mean/std)",
    }
