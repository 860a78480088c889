"""The distance facade of the drop-in API (pkg/src/elastik/engines.py:18-147).

Every call crosses the C ABI once (``ek_distance_batch``); orientation, window
selection and variant semantics follow the reference:

* ``base``        exact cost over the full matrix (no window) or the windowed
                  band with an infinite cutoff (engines.py:139-142);
* ``ea``          classic row abandoning: +inf once a whole row (left border
                  included) exceeds the cutoff, otherwise the exact cost even
                  if it is above the cutoff (_speedups.pyx:129-162);
* ``eapruned``    exact when cost <= cutoff, +inf otherwise;
* ``pruned_only`` the diagonal upper bound as a prune-only cutoff, which never
                  changes the exact result (engines.py:106-118).

An infeasible window (w < |len(s)-len(t)|) is (+inf, 0) for every windowed
variant.  ``cells_computed`` is the reference's own count for every variant
(EngineResult equality): ``base`` is lines*cols or the band; ``ea``, ``eapruned``
and ``pruned_only`` replay the reference's row logic from the GPU DP's
"value <= cutoff" masks (csrc/ek_refcells.cuh) for pairs of up to 512 columns
and 2048 rows.  Longer pairs report the band cells the GPU evaluated.
"""

from __future__ import annotations

import math
from typing import NamedTuple

import numpy as np

from . import _backend, _lib
from .errors import SpecError
from .kernels import DistanceSpec, Recurrence, make_recurrence

VARIANTS = ("base", "ea", "eapruned", "pruned_only")


class EngineResult(NamedTuple):
    cost: float
    cells_computed: int


def distance_batch(spec: DistanceSpec, variant: str, pairs, cutoffs=None, windows=None, backend=None,
                   precision: str = "float64"):
    """One GPU call for many (s, t) pairs -> (costs float64[n], cells int64[n]).

    ``pairs`` is a sequence of (s, t) series (already validated or raw);
    ``cutoffs`` per pair (default +inf); ``windows`` per pair overrides
    ``spec.window`` like the ``window`` argument of compute_ea/eapruned.
    ``precision="float32"`` runs the optional FP32 engines (costs within 1e-5
    relative of the reference; cells are the band cells the engine evaluated).
    """
    from .series import as_series

    if variant not in VARIANTS:
        raise SpecError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    _backend.resolve(backend)
    _lib.precision_code(precision)
    n = len(pairs)
    costs = np.empty(n, dtype=np.float64)
    cells = np.empty(n, dtype=np.int64)
    if n == 0:
        return costs, cells
    ss = [as_series(p[0]) for p in pairs]
    ts = [as_series(p[1]) for p in pairs]
    flat, off, lens = _lib.ragged(ss + ts)
    longest = np.maximum(lens[:n], lens[n:])
    h = _lib.SpecHandle(spec, longest_lengths=np.unique(longest), precision=precision)
    co = None
    if cutoffs is not None:
        co = np.ascontiguousarray(np.broadcast_to(np.asarray(cutoffs, dtype=np.float64), (n,)))
    wi = None
    if windows is not None:
        wi = np.ascontiguousarray(
            np.broadcast_to(np.asarray([-1 if w is None else int(w) for w in np.broadcast_to(
                np.asarray(windows, dtype=object), (n,))], dtype=np.int64), (n,)))
    so, sl, to, tl = (np.ascontiguousarray(a) for a in (off[:n], lens[:n], off[n:], lens[n:]))
    _lib.check(_lib.lib().ek_distance_batch(
        h.ref, _lib.VARIANT_CODE[variant], n, _lib.dptr(flat), len(flat), _lib.iptr(so), _lib.iptr(sl),
        _lib.iptr(to), _lib.iptr(tl), _lib.dptr(co) if co is not None else None,
        _lib.iptr(wi) if wi is not None else None, _lib.dptr(costs), _lib.iptr(cells)))
    return costs, cells


def _one(rec: Recurrence, variant: str, window, cutoff, backend) -> EngineResult:
    costs, cells = distance_batch(rec.spec, variant, [(rec.lines, rec.cols)], cutoffs=[cutoff],
                                  windows=None if window is None else [window], backend=backend)
    return EngineResult(float(costs[0]), int(cells[0]))


def _dispatch(rec: Recurrence, engine: str, window: int, cutoff: float, backend) -> EngineResult:
    """engines._dispatch (engines.py:29-50) over the GPU seam: ``_speedups.run`` semantics
    (speedups.py / ek_run_batch), the recurrence's orientation kept as built."""
    from . import speedups

    _backend.resolve(backend)
    spec = rec.spec
    h = _lib.SpecHandle(spec, longest_lengths=[max(rec.shape)])
    costs, cells = speedups._run_raw(speedups._ENGINES[engine], [rec.lines], [rec.cols], h, [int(window)],
                                     [float(cutoff)])
    return EngineResult(float(costs[0]), int(cells[0]))


def compute_base(rec: Recurrence, backend: str | None = None) -> EngineResult:
    """Exact cost over the full matrix; cells_computed is lines*cols (engines.py:60-62)."""
    return _dispatch(rec, "base", 0, math.inf, backend)


def compute_ea(rec: Recurrence, window: int, cutoff: float = math.inf, backend: str | None = None) -> EngineResult:
    """Windowed cost, abandoning once a whole row exceeds ``cutoff`` (engines.py:65-69)."""
    return _dispatch(rec, "ea", window, cutoff, backend)


def compute_eapruned(rec: Recurrence, window: int, cutoff: float = math.inf, backend: str | None = None,
                     debug: bool = False) -> EngineResult:
    """Windowed cost with pruning integrated into abandoning (engines.py:72-84).

    Exact when the true windowed cost is <= cutoff, +inf otherwise.  ``debug``
    (the reference's stale-read checker for its pure-Python row engine) has no
    GPU counterpart; use compute-sanitizer on the library instead.
    """
    return _dispatch(rec, "eapruned", window, cutoff, backend)


def diagonal_upper_bound(rec: Recurrence, window: int) -> float:
    """Cost of the diagonal-then-last-column path (engines.py:87-103).

    A host utility with the reference's summation order; the GPU engines never
    call it (pruned_only is evaluated as the exact windowed cost, which the
    bound cannot change).
    """
    from .kernels import msm_split_merge_cost, point_cost

    n_lines, n_cols = rec.shape
    if window < n_lines - n_cols:
        raise SpecError("window too small for any alignment")
    spec = rec.spec
    mode = spec.cost_mode
    lv, cv = rec.lines.tolist(), rec.cols.tolist()

    def canonical(i, j):
        if spec.kind in ("dtw", "cdtw", "erp"):
            return point_cost(lv[i - 1], cv[j - 1], mode)
        if spec.kind == "wdtw":
            return point_cost(lv[i - 1], cv[j - 1], mode) * rec.wdtw_weights[abs(i - j)]
        if spec.kind == "msm":
            return abs(lv[i - 1] - cv[j - 1])
        sp = lv[i - 2] if i >= 2 else 0.0
        tp = cv[j - 2] if j >= 2 else 0.0
        dij = float(abs(i - j))
        return point_cost(lv[i - 1], cv[j - 1], mode) + point_cost(sp, tp, mode) + spec.twe_nu * (dij + dij)

    def alt_row(i, j):
        if spec.kind == "erp":
            return point_cost(lv[i - 1], spec.erp_gap, mode)
        if spec.kind == "msm":
            return msm_split_merge_cost(lv[i - 1], lv[i - 2] if i >= 2 else lv[i - 1], cv[j - 1], spec.msm_c)
        if spec.kind == "twe":
            return point_cost(lv[i - 1], lv[i - 2] if i >= 2 else 0.0, mode) + spec.twe_nu + spec.twe_lambda
        return canonical(i, j)

    total = rec.init_corner
    for k in range(1, n_cols + 1):
        total += canonical(k, k)
    for i in range(n_cols + 1, n_lines + 1):
        total += alt_row(i, n_cols)
    return total


def compute_pruned_only(rec: Recurrence, window: int, backend: str | None = None) -> EngineResult:
    """Exact windowed cost; never abandons on a feasible window (engines.py:106-118)."""
    return _one(rec, "pruned_only", window, math.inf, backend)


def distance(spec: DistanceSpec, variant: str, s, t, cutoff: float = math.inf,
             backend: str | None = None) -> EngineResult:
    """``spec`` between ``s`` and ``t`` with the named variant (engines.py:121-147)."""
    if variant not in VARIANTS:
        raise SpecError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    rec = make_recurrence(spec, s, t)
    if variant == "base":
        if spec.window is None:
            return compute_base(rec, backend=backend)
        return _one(rec, "base", spec.window, math.inf, backend)
    window = spec.effective_window(len(rec.lines))
    if variant == "ea":
        return compute_ea(rec, window, cutoff, backend=backend)
    if variant == "eapruned":
        return compute_eapruned(rec, window, cutoff, backend=backend)
    return compute_pruned_only(rec, window, backend=backend)
