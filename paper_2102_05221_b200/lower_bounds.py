"""Envelopes and LB_Keogh bounds of the drop-in API (lower_bounds.py:1-98).

Host utilities with the reference's exact semantics.  The GPU search paths build
their own FP32 envelopes and bounds on the device (csrc/ek_lb.cuh, ek_subseq.cuh);
these functions exist for callers of the reference API (e.g. ``nn_search``'s
``envelopes=`` argument) and give bit-identical values to the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionError
from .series import as_series


@dataclass(frozen=True)
class Envelope:
    """Running max / min of a series over [i - window, i + window]."""

    upper: np.ndarray
    lower: np.ndarray
    window: int


def _sliding(s: np.ndarray, window: int, op) -> np.ndarray:
    """op-reduction of s over [i - w, i + w] (clipped): a doubling table of runs of
    2^k, then two overlapping runs per point -- max/min select values, so the result
    is exactly the reference's deque output."""
    n = len(s)
    span = 2 * window + 1
    if span >= 2 * n - 1:  # every window covers the whole series
        return np.full(n, op.reduce(s))
    pad = np.concatenate([np.full(window, s[0]), s, np.full(window, s[-1])])
    # runs of length 2^k starting at every position of the padded series
    tables = [pad]
    length = 1
    while 2 * length <= span:
        prev = tables[-1]
        tables.append(op(prev[:-length], prev[length:]))
        length *= 2
    run = tables[-1]
    return op(run[:n], run[span - length: span - length + n])


def build_envelope(s, window: int) -> Envelope:
    """Envelope of s for a +-window band (lower_bounds.py:23-57)."""
    s = as_series(s)
    if window < 0:
        raise ValueError("window must be >= 0")
    w = min(int(window), len(s))
    return Envelope(upper=_sliding(s, w, np.maximum), lower=_sliding(s, w, np.minimum), window=window)


def lb_keogh(q, env: Envelope, cost_mode: str = "squared") -> float:
    """Sum over points of the distance from q to the envelope (lower_bounds.py:60-84),
    accumulated left to right like the reference."""
    q = as_series(q)
    if len(q) != len(env.upper):
        raise DimensionError(f"query length {len(q)} does not match envelope length {len(env.upper)}")
    above = q > env.upper
    below = q < env.lower
    d = np.where(above, q - env.upper, np.where(below, env.lower - q, 0.0))
    terms = d * d if cost_mode == "squared" else d
    terms = terms[above | below]
    if terms.size == 0:
        return 0.0
    return float(np.add.accumulate(terms)[-1])  # sequential, starting from the first term


def lb_keogh2(q, c, env_c: Envelope, env_q: Envelope, cutoff: float = np.inf,
              cost_mode: str = "squared") -> float:
    """max(lb_keogh(q, env_c), lb_keogh(c, env_q)); the second only when the first is
    <= cutoff (lower_bounds.py:87-98)."""
    first = lb_keogh(q, env_c, cost_mode)
    if first > cutoff:
        return first
    second = lb_keogh(c, env_q, cost_mode)
    return max(first, second) if second > first else first


def build_envelopes(batch, window: int) -> list[Envelope]:
    """build_envelope for a batch of equal-length series in one GPU call
    (csrc/ek_misc.cu k_envelope, exact double tables); same values as the host
    function and the reference.  Raises DimensionError for ragged batches."""
    from . import _lib
    from .search import _pack

    if window < 0:
        raise ValueError("window must be >= 0")
    flat, off, lens = _pack(batch)
    n = len(lens)
    if n == 0:
        return []
    if np.any(lens != lens[0]):
        raise DimensionError("build_envelopes needs series of one length")
    length = int(lens[0])
    up = np.empty((n, length), dtype=np.float64)
    lo = np.empty((n, length), dtype=np.float64)
    L = _lib.lib()
    _lib.check(L.ek_envelopes(_lib.dptr(flat), len(flat), _lib.iptr(off), n, length, int(window), _lib.dptr(up),
                              _lib.dptr(lo)))
    return [Envelope(upper=up[k], lower=lo[k], window=window) for k in range(n)]
