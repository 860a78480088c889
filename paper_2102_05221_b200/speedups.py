"""GPU drop-in for the reference's native module ``elastik._speedups``.

The reference's one native seam is ``_speedups.run`` (pkg/src/elastik/_speedups.pyx:274-317),
called once per pair by ``engines._dispatch`` (pkg/src/elastik/engines.py:29-50) with the
payload ``make_recurrence`` built (kernels.py:157-277).  This module exports the same
names -- ``EMPTY`` and ``run`` with the same positional signature, engine names, argument
meaning and return value -- computed on the GPU through ``ek_run_batch``
(include/elastik_b200.h).  A maintainer plugs it in by letting ``_backend.speedups()``
return this module for ``backend="cuda"`` (path B); ``_dispatch`` is then
unchanged.  ``run_many`` is the batched form (one GPU call for many pairs).

Semantics of ``run`` (the reference's, kept exactly):

* ``engine`` is ``"base"``, ``"ea"`` or ``"eapruned"`` (a ``KeyError`` otherwise, like the
  ``_ENGINES[engine]`` lookup of the .pyx);
* ``lines`` / ``cols`` are used as given -- no re-orientation;
* ``base`` is the full matrix: ``window`` and ``cutoff`` are ignored and cells = nl*nc;
* ``ea`` / ``eapruned`` use ``window`` and ``cutoff``; an infeasible window
  (``window < nl - nc``) is ``(inf, 0)``;
* the return value is ``(cost, cells_computed)``.

Payload arrays: ``weights`` is the WDTW table ``make_recurrence`` passes (length
max(nl, nc) + 1, host libm ``exp``); it is uploaded as given.  ``vborder_vals`` /
``hborder_vals`` are ERP's cumulative gap borders (``kernels._erp_border``), which the GPU
engines rebuild bit-identically from the series; any other border payload (non-ERP kinds
with borders, or ERP without them) is not what ``make_recurrence`` produces and raises
``NotImplementedError`` instead of computing something else.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .kernels import KINDS

EMPTY = np.empty(0, dtype=np.float64)
EMPTY.setflags(write=False)

_ENGINES = {"base": 0, "ea": 1, "eapruned": 2}


def _vec(a, name):
    """``const double[::1]``: a C-contiguous 1-D float64 buffer (no conversion, like Cython)."""
    if not isinstance(a, np.ndarray):
        a = np.asarray(memoryview(a))
    if a.dtype != np.float64:
        raise ValueError(f"Buffer dtype mismatch, expected 'const double' but got '{a.dtype}' for {name}")
    if a.ndim != 1:
        raise ValueError(f"Buffer has wrong number of dimensions (expected 1, got {a.ndim}) for {name}")
    if not a.flags.c_contiguous:
        raise ValueError(f"ndarray is not C-contiguous ({name})")
    return a


def _pc(x, g, mode):
    d = x - g
    return d * d if mode == 0 else np.abs(d)


def _check_borders(kind, mode, lines, cols, gap, vb, hb):
    """The payload must be what make_recurrence builds (see the module docstring)."""
    if kind != KINDS.index("erp"):
        if len(vb) or len(hb):
            raise NotImplementedError("border payloads are only defined for erp (kernels.py:244-262)")
        return
    if len(vb) != len(lines) + 1 or len(hb) != len(cols) + 1:
        raise NotImplementedError("erp needs the cumulative gap borders of kernels._erp_border")
    # _erp_border: sequential prefix sums (np.add.accumulate is a sequential loop)
    want_v = np.add.accumulate(_pc(lines, gap, mode))
    want_h = np.add.accumulate(_pc(gap, cols, mode))
    if vb[0] != 0.0 or hb[0] != 0.0 or not (np.array_equal(vb[1:], want_v) and np.array_equal(hb[1:], want_h)):
        raise NotImplementedError("erp border payload differs from kernels._erp_border; custom borders are "
                                  "not supported by the GPU engines")


class _RunSpec:
    """ek_spec for run's scalar arguments; WDTW tables come from the caller's payload."""

    def __init__(self, kind, mode, erp_gap, msm_c, twe_nu, twe_lambda, tables):
        self._keep = []
        tabs = offs = None
        mx = 0
        if tables:
            mx = max(tables)
            offs = np.full(mx + 1, -1, dtype=np.int64)
            parts, pos = [], 0
            for m in sorted(tables):
                offs[m] = pos
                parts.append(tables[m])
                pos += m + 1
            tabs = np.ascontiguousarray(np.concatenate(parts))
            self._keep += [tabs, offs]
        self.s = _lib.EkSpec(int(kind), int(mode), -1, float(erp_gap), float(msm_c), float(twe_nu),
                             float(twe_lambda), _lib.dptr(tabs) if tabs is not None else None,
                             _lib.iptr(offs) if offs is not None else None, mx, 0)

    @property
    def ref(self):
        import ctypes

        return ctypes.byref(self.s)


def run_many(engine, pairs, kind, mode, windows, cutoffs, erp_gap, msm_c, twe_nu, twe_lambda,
             weights=None, borders=None):
    """``run`` for many pairs in one GPU call.

    ``pairs``: sequence of (lines, cols); ``windows`` / ``cutoffs``: scalars or one per pair;
    ``weights``: per-pair WDTW tables (or one shared table / None); ``borders``: per-pair
    (vborder_vals, hborder_vals) or None.  Returns (costs float64[n], cells int64[n]).
    """
    code = _ENGINES[engine]
    kind, mode = int(kind), int(mode)
    if not 0 <= kind < len(KINDS):
        raise ValueError(f"kind code {kind} out of range")
    if mode not in (0, 1):
        raise ValueError(f"mode code {mode} out of range")
    n = len(pairs)
    costs = np.empty(n, dtype=np.float64)
    cells = np.empty(n, dtype=np.int64)
    if n == 0:
        return costs, cells
    lines = [_vec(p[0], "lines") for p in pairs]
    cols = [_vec(p[1], "cols") for p in pairs]
    for k in range(n):
        if len(lines[k]) == 0 or len(cols[k]) == 0:
            raise ValueError("run needs non-empty series (make_recurrence's as_series guarantees it)")
        if not (np.isfinite(lines[k]).all() and np.isfinite(cols[k]).all()):
            raise ValueError("time series values must all be finite")
    tables = {}
    if kind == KINDS.index("wdtw"):
        for k in range(n):
            wt = weights[k] if isinstance(weights, (list, tuple)) else weights
            if wt is None or len(wt) == 0:
                raise ValueError("wdtw needs its weight table (kernels.wdtw_weight_table)")
            wt = _vec(wt, "weights")
            m = max(len(lines[k]), len(cols[k]))
            if len(wt) != m + 1:
                raise ValueError(f"wdtw weight table has {len(wt)} entries, expected max(nl, nc) + 1 = {m + 1}")
            if m in tables and not np.array_equal(tables[m], wt):
                raise NotImplementedError("different wdtw tables for the same length in one batch")
            tables[m] = wt
    for k in range(n):
        vb, hb = borders[k] if borders is not None else (EMPTY, EMPTY)
        _check_borders(kind, mode, lines[k], cols[k], float(erp_gap), _vec(vb, "vborder_vals"),
                       _vec(hb, "hborder_vals"))
    return _run_raw(code, lines, cols, _RunSpec(kind, mode, erp_gap, msm_c, twe_nu, twe_lambda, tables), windows,
                    cutoffs)


def _run_raw(code, lines, cols, h, windows, cutoffs):
    """ek_run_batch over validated, oriented pairs (also the compute_* facade's path)."""
    n = len(lines)
    costs = np.empty(n, dtype=np.float64)
    cells = np.empty(n, dtype=np.int64)
    flat, off, lens = _lib.ragged(list(lines) + list(cols))
    wi = np.ascontiguousarray(np.broadcast_to(np.asarray(windows, dtype=np.int64), (n,)))
    co = np.ascontiguousarray(np.broadcast_to(np.asarray(cutoffs, dtype=np.float64), (n,)))
    lo, ll, cof, cl = (np.ascontiguousarray(a) for a in (off[:n], lens[:n], off[n:], lens[n:]))
    _lib.check(_lib.lib().ek_run_batch(h.ref, code, n, _lib.dptr(flat), len(flat), _lib.iptr(lo), _lib.iptr(ll),
                                       _lib.iptr(cof), _lib.iptr(cl), _lib.iptr(wi), _lib.dptr(co),
                                       _lib.dptr(costs), _lib.iptr(cells)))
    return costs, cells


def run(engine, lines, cols, kind, mode, window, cutoff, erp_gap, msm_c, twe_nu, twe_lambda, weights,
        vborder_vals, hborder_vals):
    """Run one engine over raw arrays; returns (cost, cells_computed) (_speedups.pyx:274-317)."""
    costs, cells = run_many(engine, [(lines, cols)], kind, mode, [int(window)], [float(cutoff)], erp_gap, msm_c,
                            twe_nu, twe_lambda, weights=[weights], borders=[(vborder_vals, hborder_vals)])
    return float(costs[0]), int(cells[0])


__all__ = ["EMPTY", "run", "run_many"]
