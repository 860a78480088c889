"""Series validation and the dataset container of the drop-in API.

``as_series`` is the validating constructor every public entry point applies
before crossing the C ABI (pkg/src/elastik/series.py:19-31).  ``znormalize`` is
kept as a host utility with the reference's numpy semantics
(series.py:118-131); the subsequence-search hot path normalises windows on the
GPU (csrc/ek_subseq.cuh) and never calls it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DegenerateInputError, EmptyDatasetError


def as_series(values) -> np.ndarray:
    """Contiguous 1-D float64 array, length >= 1, all finite; ValueError otherwise."""
    arr = np.ascontiguousarray(values, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError(f"time series must be 1-D, got shape {arr.shape}")
    if arr.size < 1:
        raise ValueError("time series must contain at least one value")
    if not np.isfinite(arr).all():
        raise ValueError("time series values must all be finite")
    return arr


@dataclass(frozen=True)
class LabeledDataset:
    """(integer label, series) pairs; lengths may differ (series.py:34-58)."""

    name: str
    entries: tuple

    def __post_init__(self):
        if not self.entries:
            raise EmptyDatasetError(f"dataset {self.name!r} has no entries")

    def __len__(self):
        return len(self.entries)

    @property
    def labels(self) -> list[int]:
        return [label for label, _ in self.entries]

    @property
    def series(self) -> list[np.ndarray]:
        return [values for _, values in self.entries]


def znormalize(s) -> np.ndarray:
    """Mean 0 / population std 1; std < 1e-12 -> zeros; needs length >= 2."""
    s = np.asarray(s, dtype=np.float64)
    if s.size < 2:
        raise DegenerateInputError("z-normalization needs at least 2 points")
    mean = s.mean()
    std = s.std()
    if std < 1e-12:
        return np.zeros_like(s)
    return (s - mean) / std
