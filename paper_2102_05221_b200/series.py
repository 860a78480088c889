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

from .errors import DegenerateInputError, EmptyDatasetError, ParseError


def as_series(values, finite_on_device: bool = False) -> np.ndarray:
    """Contiguous 1-D float64 array, length >= 1, all finite; ValueError otherwise.

    ``finite_on_device``: the caller hands the array to a library entry that checks
    finiteness on the GPU after the upload and reports the same ValueError (ek_subseq,
    ek_subseq_profile: csrc/ek_api.cu inputs_finite), so a long stream is not scanned twice.
    """
    arr = np.ascontiguousarray(values, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError(f"time series must be 1-D, got shape {arr.shape}")
    if arr.size < 1:
        raise ValueError("time series must contain at least one value")
    if not (finite_on_device and arr.size >= 4096) and not np.isfinite(arr).all():
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


# ---- ingestion: UCR-format text files, derivative, generator ----------

_SEPARATORS = {"tab": "\t", "comma": ","}


def _separator(delimiter: str) -> str:
    if delimiter not in _SEPARATORS:
        raise ValueError(f"delimiter must be one of {sorted(_SEPARATORS)}, got {delimiter!r}")
    return _SEPARATORS[delimiter]


def _number(token: str, line: int, column: int) -> float:
    try:
        x = float(token)
    except ValueError:
        raise ParseError(f"not a number: {token!r}", line, column) from None
    if x != x or x in (float("inf"), float("-inf")):
        raise ParseError(f"non-finite value: {token!r}", line, column)
    return x


def load_tsv(path, delimiter: str = "tab", name: str | None = None) -> LabeledDataset:
    """UCR-format dataset (series.py:61-86): one series per line, the (numeric, truncated
    to int) label first; tab or comma separated; LF or CRLF; blank lines skipped.
    Malformed fields raise ParseError with their 1-based line and column."""
    sep = _separator(delimiter)
    entries = []
    with open(path, "r", encoding="utf-8") as fh:
        for line_no, text in enumerate(fh, start=1):
            text = text.rstrip("\r\n")
            if not text.strip():
                continue
            parts = text.split(sep)
            if len(parts) < 2:
                raise ParseError("expected a label and at least one value", line_no, 1)
            label = int(_number(parts[0], line_no, 1))
            values = np.array([_number(tok, line_no, k) for k, tok in enumerate(parts[1:], start=2)],
                              dtype=np.float64)
            entries.append((label, values))
    if not entries:
        raise EmptyDatasetError(f"no series found in {path}")
    return LabeledDataset(name=str(path) if name is None else name, entries=tuple(entries))


def write_tsv(dataset: LabeledDataset, path, delimiter: str = "tab") -> None:
    """Inverse of load_tsv (series.py:89-98); repr() keeps a reload bit-identical."""
    sep = _separator(delimiter)
    with open(path, "w", encoding="utf-8") as fh:
        for label, values in dataset.entries:
            fh.write(sep.join([str(int(label))] + [repr(float(v)) for v in values]) + "\n")


def derivative(s) -> np.ndarray:
    """First-derivative transform (series.py:134-144), two points shorter:
    out[i] = ((s[i+1] - s[i]) + (s[i+2] - s[i]) / 2) / 2, in that operation order."""
    s = np.asarray(s, dtype=np.float64)
    if s.size < 3:
        raise DegenerateInputError("derivative transform needs at least 3 points")
    step = s[1:-1] - s[:-2]
    slope = (s[2:] - s[:-2]) / 2.0
    return (step + slope) / 2.0


def gen_random_walk(count: int, length: int, classes: int, seed: int, name: str = "random-walk",
                    drift_step: float = 0.15) -> LabeledDataset:
    """Labelled random walks (series.py:147-170): label = index mod classes; the walk of
    class k steps N(drift_step * (k - (classes-1)/2), 1), one rng.normal draw of `length`
    per series from default_rng(seed), cumulated."""
    if min(count, length, classes) < 1:
        raise ValueError("count, length and classes must all be >= 1")
    rng = np.random.default_rng(seed)
    entries = []
    centre = (classes - 1) / 2.0
    for k in range(count):
        label = k % classes
        walk = np.cumsum(rng.normal(loc=drift_step * (label - centre), scale=1.0, size=length))
        entries.append((label, walk))
    return LabeledDataset(name=name, entries=tuple(entries))
