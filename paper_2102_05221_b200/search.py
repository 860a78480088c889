"""1-NN search, 1-NN classification, subsequence search and all-pairs matrices.

Drop-in counterparts of pkg/src/elastik/search.py:25-215.  The reference scans
candidates serially, one ``distance()`` call per pair with the running best as
the cutoff.  Here one C-ABI call hands the whole query batch to the GPU
(``ek_nn`` / ``ek_subseq`` / ``ek_pairwise``): every pair is evaluated with a
per-query shared cutoff that only tightens, so each result is either exact or
+inf, and a lexicographic (distance, index) reduction returns the reference's
answer -- ties keep the lowest candidate index / offset -- whatever the
schedule ("1-NN ties").

Results (distance, index, label, offset) are identical to the reference for
every variant and lower-bound mode.  The accounting in ``SearchStats``
(computed / abandoned / cells) describes the GPU schedule; ``lb_skips`` is 0
(the lower-bound pre-filters are a ranked "next" item, SURVEY.md 8(f)#1, and
cannot change results), and ``trace`` stays empty (there is no serial cutoff
sequence to trace).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _backend, _lib
from .engines import VARIANTS
from .errors import DegenerateInputError, DimensionError, SearchError, SpecError
from .kernels import DistanceSpec
from .series import LabeledDataset, as_series

LB_MODES = ("none", "keogh", "keogh2")


@dataclass(frozen=True)
class SearchConfig:
    """Distance, engine variant and lower-bound mode for one search run (search.py:25-42)."""

    spec: DistanceSpec
    variant: str = "eapruned"
    lb: str = "none"
    normalize: bool = False
    debug: bool = False
    backend: str | None = None
    # not in the reference: "float32" selects the optional FP32 engines for nn_search /
    # classify_1nn (distances within 1e-5 relative; near-ties may pick another index)
    precision: str = "float64"

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise SpecError(f"unknown variant {self.variant!r}; expected one of {VARIANTS}")
        if self.lb not in LB_MODES:
            raise SpecError(f"unknown lb mode {self.lb!r}; expected one of {LB_MODES}")
        if self.lb != "none" and self.spec.kind not in ("dtw", "cdtw"):
            raise SpecError("lower bounds are only available for dtw and cdtw")
        _lib.precision_code(self.precision)


@dataclass
class SearchStats:
    """Per-query accounting; lb_skips + computed + abandoned == candidates seen."""

    computed: int = 0
    abandoned: int = 0
    lb_skips: int = 0
    cells: int = 0
    wall_time: float = 0.0
    trace: list = field(default_factory=list)


@dataclass(frozen=True)
class SearchRecord:
    """One classified query, as reported by :func:`classify_1nn`."""

    query_index: int
    actual: int
    predicted: int
    nn_index: int
    nn_distance: float
    computed: int
    abandoned: int
    lb_skips: int
    cells: int
    wall_time: float


def _pack(series):
    """Series collection -> (flat float64, offsets, lengths).  A 2-D C-contiguous float64
    array (equal lengths) is used in place -- no copy, so a pinned host array stays
    pinned for the library's host-to-device copy, and the library checks finiteness on
    the device; anything else goes through as_series per series (the reference's
    validation) and is concatenated."""
    if isinstance(series, np.ndarray) and series.ndim == 2 and series.dtype == np.float64 \
            and series.flags.c_contiguous:
        n, length = series.shape
        if n and length < 1:
            raise ValueError("time series must contain at least one value")
        # finiteness is checked by the library on the uploaded copy (ValueError, same message)
        return series.reshape(-1), np.arange(n, dtype=np.int64) * length, np.full(n, length, dtype=np.int64)
    return _lib.ragged([as_series(x) for x in series])


def _nn_prepare(spec: DistanceSpec, variant: str, queries, candidates, backend, precision: str):
    """Validation and packing shared by nn_batch and NNPipeline: (args of ek_nn up to the
    outputs, the output arrays, the objects those pointers point into)."""
    _backend.resolve(backend)
    _lib.precision_code(precision)
    if variant not in VARIANTS:
        raise SpecError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    qf, qo, ql = _pack(queries)
    cf, co, cl = _pack(candidates)
    if len(cl) == 0:
        raise SearchError("candidate set is empty")
    nq = len(ql)
    out = [np.empty(nq, dtype=np.int64), np.empty(nq, dtype=np.float64)] + [np.empty(nq, dtype=np.int64)
                                                                             for _ in range(3)]
    if spec.kind == "wdtw":
        longest = np.unique(np.maximum.outer(np.unique(ql), np.unique(cl))) if nq else ()
    else:
        longest = ()  # only WDTW needs per-length tables
    h = _lib.SpecHandle(spec, longest_lengths=longest, precision=precision)
    args = (h.ref, _lib.VARIANT_CODE[variant], _lib.dptr(qf), len(qf), _lib.iptr(qo), _lib.iptr(ql), nq,
            _lib.dptr(cf), len(cf), _lib.iptr(co), _lib.iptr(cl), len(cl))
    return args, out, (h, qf, qo, ql, cf, co, cl)


def nn_batch(spec: DistanceSpec, variant: str, queries, candidates, backend=None, precision: str = "float64"):
    """1-NN of every query in one GPU call.

    Returns arrays (nn_index int64, nn_distance float64, cells, computed,
    abandoned); nn_index is -1 when every candidate is +inf.  ``precision``
    "float32" runs the optional FP32 engines.
    """
    args, out, _keep = _nn_prepare(spec, variant, queries, candidates, backend, precision)
    if len(out[0]) == 0:
        return tuple(out)
    L = _lib.lib()
    _lib.check(L.ek_nn(*args, _lib.iptr(out[0]), _lib.dptr(out[1]), _lib.iptr(out[2]), _lib.iptr(out[3]),
                       _lib.iptr(out[4])))
    return tuple(out)


class NNPipeline:
    """nn_batch over a stream of batches, two deep (ek_nn_submit / ek_nn_collect).

    ``submit(queries, candidates)`` enqueues a batch and returns at once; ``collect()``
    returns the oldest batch's ``nn_batch`` tuple.  At most two batches are in flight, so
    batch k+1's host-to-device upload overlaps batch k's search.  The inputs must not be
    modified until their batch is collected (page-locked arrays, e.g. ingest's packed
    batches, make the upload asynchronous).  Results and errors equal nn_batch's.
    """

    DEPTH = 2

    def __init__(self, spec: DistanceSpec, variant: str, backend=None, precision: str = "float64"):
        self.spec, self.variant, self.backend, self.precision = spec, variant, backend, precision
        self._inflight = []  # (slot, out, keep) in submission order
        self._next = 0

    def __len__(self):
        return len(self._inflight)

    def submit(self, queries, candidates) -> None:
        if len(self._inflight) >= self.DEPTH:
            raise SearchError(f"NNPipeline: {self.DEPTH} batches in flight; collect() first")
        args, out, keep = _nn_prepare(self.spec, self.variant, queries, candidates, self.backend, self.precision)
        if len(out[0]) == 0:
            self._inflight.append((None, out, keep))
            return
        slot = self._next
        _lib.check(_lib.lib().ek_nn_submit(*args, slot))
        self._next ^= 1
        self._inflight.append((slot, out, keep))

    def collect(self):
        if not self._inflight:
            raise SearchError("NNPipeline: nothing submitted")
        slot, out, _keep = self._inflight.pop(0)
        if slot is not None:
            _lib.check(_lib.lib().ek_nn_collect(slot, _lib.iptr(out[0]), _lib.dptr(out[1]), _lib.iptr(out[2]),
                                                _lib.iptr(out[3]), _lib.iptr(out[4])))
        return tuple(out)

    def drain(self):
        """Collect (and drop) whatever is still in flight, e.g. after an error."""
        while self._inflight:
            try:
                self.collect()
            except Exception:  # noqa: BLE001 -- draining after a failure
                pass


def nn_batch_stream(spec: DistanceSpec, variant: str, batches, backend=None, precision: str = "float64"):
    """Yield nn_batch(spec, variant, Q, C) for every (Q, C) of ``batches``, in order, with the
    next batch's upload overlapping the current batch's search (NNPipeline)."""
    pipe = NNPipeline(spec, variant, backend=backend, precision=precision)
    try:
        for q, c in batches:
            if len(pipe) == NNPipeline.DEPTH:
                yield pipe.collect()
            pipe.submit(q, c)
        while len(pipe):
            yield pipe.collect()
    finally:
        pipe.drain()


def nn_search(query, candidates, cfg: SearchConfig, envelopes=None):
    """Nearest neighbour of ``query`` -> ``(distance, index, stats)`` (search.py:81-125)."""
    query = as_series(query)
    candidates = list(candidates)
    if not candidates:
        raise SearchError("candidate set is empty")
    start = time.perf_counter()
    idx, dist, cells, comp, ab = nn_batch(cfg.spec, cfg.variant, [query], candidates, backend=cfg.backend,
                                          precision=cfg.precision)
    stats = SearchStats(computed=int(comp[0]), abandoned=int(ab[0]), cells=int(cells[0]))
    stats.wall_time = time.perf_counter() - start
    return float(dist[0]), int(idx[0]), stats


def _batch(ds):
    """The series of a LabeledDataset, or of an ingest.PackedDataset: equal lengths as a 2-D
    view of its (page-locked) buffer, which ek_nn uploads without a copy."""
    from .ingest import PackedDataset

    if isinstance(ds, PackedDataset):
        n = len(ds)
        if n and np.all(ds.lengths == ds.lengths[0]) and np.array_equal(ds.offsets, np.arange(n) * ds.lengths[0]):
            return ds.values[:n * int(ds.lengths[0])].reshape(n, int(ds.lengths[0]))
        return [ds.series(s) for s in range(n)]
    return ds.series


def classify_1nn(train: LabeledDataset, test: LabeledDataset, cfg: SearchConfig,
                 threads: int | None = None) -> list[SearchRecord]:
    """1-NN classification of every test series against the train set (search.py:128-160).

    All queries go to the GPU in one call; ``threads`` is accepted for
    signature compatibility and has no effect.  ``train`` / ``test`` may also be
    ``ingest.PackedDataset`` batches (load_tsv_packed).
    """
    labels = [int(x) for x in train.labels]
    start = time.perf_counter()
    idx, dist, cells, comp, ab = nn_batch(cfg.spec, cfg.variant, _batch(test), _batch(train), backend=cfg.backend,
                                          precision=cfg.precision)
    per_query = (time.perf_counter() - start) / max(1, len(test))
    records = []
    for q, actual in enumerate(int(x) for x in test.labels):
        best = int(idx[q])
        records.append(SearchRecord(
            query_index=q, actual=actual, predicted=labels[best] if best >= 0 else -1, nn_index=best,
            nn_distance=float(dist[q]), computed=int(comp[q]), abandoned=int(ab[q]), lb_skips=0,
            cells=int(cells[q]), wall_time=per_query))
    return records


def subsequence_search(query, reference, cfg: SearchConfig):
    """Best-matching window of ``reference`` -> ``(offset, distance, stats)`` (search.py:163-215).

    Windows (and the query) are z-normalised on the GPU with numpy's exact
    arithmetic when ``cfg.normalize``; ties keep the lowest offset.
    """
    if cfg.spec.kind not in ("dtw", "cdtw"):
        raise SpecError("subsequence search supports dtw and cdtw only")
    if cfg.precision != "float64":
        raise SpecError("subsequence search runs in float64 only")
    query = as_series(query)
    reference = as_series(reference, finite_on_device=True)  # the library validates the uploaded stream
    lq = len(query)
    if lq > len(reference):
        raise DimensionError(f"query length {lq} exceeds reference length {len(reference)}")
    if cfg.normalize and lq < 2:
        raise DegenerateInputError("z-normalization needs at least 2 points")
    _backend.resolve(cfg.backend)
    h = _lib.SpecHandle(cfg.spec)
    off = np.zeros(1, dtype=np.int64)
    dist = np.zeros(1, dtype=np.float64)
    cells = np.zeros(1, dtype=np.int64)
    comp = np.zeros(1, dtype=np.int64)
    ab = np.zeros(1, dtype=np.int64)
    start = time.perf_counter()
    _lib.check(_lib.lib().ek_subseq(h.ref, _lib.VARIANT_CODE[cfg.variant], _lib.dptr(query), lq,
                                    _lib.dptr(reference), len(reference), int(bool(cfg.normalize)), _lib.iptr(off),
                                    _lib.dptr(dist), _lib.iptr(cells), _lib.iptr(comp), _lib.iptr(ab)))
    stats = SearchStats(computed=int(comp[0]), abandoned=int(ab[0]), cells=int(cells[0]))
    stats.wall_time = time.perf_counter() - start
    return int(off[0]), float(dist[0]), stats


def subsequence_profile(query, reference, spec: DistanceSpec, normalize: bool = False, backend=None):
    """Distance of ``query`` to every stride-1 window of ``reference`` (variant "base").

    Entry ``o`` equals ``distance(spec, "base", query, reference[o:o+lq])`` with both
    sides z-normalised when ``normalize`` -- the per-offset values subsequence_search
    (search.py:189-213) compares, without its running cutoff.
    """
    if spec.kind not in ("dtw", "cdtw"):
        raise SpecError("subsequence search supports dtw and cdtw only")
    query = as_series(query)
    reference = as_series(reference, finite_on_device=True)  # the library validates the uploaded stream
    lq = len(query)
    if lq > len(reference):
        raise DimensionError(f"query length {lq} exceeds reference length {len(reference)}")
    if normalize and lq < 2:
        raise DegenerateInputError("z-normalization needs at least 2 points")
    _backend.resolve(backend)
    h = _lib.SpecHandle(spec)
    out = np.empty(len(reference) - lq + 1, dtype=np.float64)
    _lib.check(_lib.lib().ek_subseq_profile(h.ref, _lib.dptr(query), lq, _lib.dptr(reference), len(reference),
                                            int(bool(normalize)), _lib.dptr(out)))
    return out


def pairwise(spec: DistanceSpec, X, variant: str = "pruned_only", backend=None, precision: str = "float64"):
    """Full symmetric matrix of ``distance(spec, variant, X[i], X[j])``, diagonal 0.0.

    The all-pairs loop of SURVEY.md 3.4 in one GPU call; d(a,b) == d(b,a)
    bit-exactly, so the upper triangle is evaluated and mirrored.  Returns
    ``(D, cells)``.  ``precision="float32"``: the optional FP32 engines.
    """
    if variant not in VARIANTS:
        raise SpecError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    _backend.resolve(backend)
    _lib.precision_code(precision)
    flat, off, lens = _pack(X)
    n = len(lens)
    D = np.zeros((n, n), dtype=np.float64)
    if n == 0:
        return D, 0
    longest = np.unique(np.maximum.outer(np.unique(lens), np.unique(lens)))
    h = _lib.SpecHandle(spec, longest_lengths=longest, precision=precision)
    cells = np.zeros(1, dtype=np.int64)
    _lib.check(_lib.lib().ek_pairwise(h.ref, _lib.VARIANT_CODE[variant], _lib.dptr(flat), len(flat),
                                      _lib.iptr(off), _lib.iptr(lens), n, _lib.dptr(D), _lib.iptr(cells)))
    return D, int(cells[0])


def pairwise_range(spec: DistanceSpec, X, pair_lo: int, pair_hi: int, variant: str = "pruned_only", backend=None,
                   precision: str = "float64"):
    """Pairs [pair_lo, pair_hi) of the upper triangle, in ``numpy.triu_indices(n, 1)`` order,
    in one GPU call -> (costs float64[pair_hi - pair_lo], cells).  The all-pairs shard of a
    rank (distributed.pairwise_sharded); the device maps pair indices to (i, j)."""
    if variant not in VARIANTS:
        raise SpecError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    _backend.resolve(backend)
    _lib.precision_code(precision)
    flat, off, lens = _pack(X)
    n = len(lens)
    total = n * (n - 1) // 2
    if not 0 <= pair_lo <= pair_hi <= total:
        raise ValueError(f"pair range [{pair_lo}, {pair_hi}) outside [0, {total})")
    out = np.empty(pair_hi - pair_lo, dtype=np.float64)
    if pair_hi == pair_lo:
        return out, 0
    longest = np.unique(np.maximum.outer(np.unique(lens), np.unique(lens)))
    h = _lib.SpecHandle(spec, longest_lengths=longest, precision=precision)
    cells = np.zeros(1, dtype=np.int64)
    _lib.check(_lib.lib().ek_pairwise_range(h.ref, _lib.VARIANT_CODE[variant], _lib.dptr(flat), len(flat),
                                            _lib.iptr(off), _lib.iptr(lens), n, int(pair_lo), int(pair_hi),
                                            _lib.dptr(out), _lib.iptr(cells)))
    return out, int(cells[0])


_ = math  # re-exported names only
