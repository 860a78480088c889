"""Drive the reference's OWN compiled kernel -- TEST / BASELINE INFRASTRUCTURE ONLY.

``oracle/_ref/_speedups*.so`` is built by ``oracle/Makefile`` straight from
``/root/reference/pkg/src/elastik/_speedups.pyx`` with the reference's flags.
The reference's Python glue cannot travel to the GPU box (``/root/reference``
does not exist there), so this module restates it around that compiled
kernel:

* payload construction of ``make_recurrence`` (pkg/src/elastik/kernels.py:157-277):
  orientation, WDTW table (``math.exp``), ERP cumulative borders;
* ``_dispatch`` argument marshalling (pkg/src/elastik/engines.py:29-50);
* the variant facade incl. ``diagonal_upper_bound`` (engines.py:87-147);
* ``nn_search`` (search.py:81-125), the all-pairs loop, ``subsequence_search``
  (search.py:163-215) with numpy ``znormalize`` (series.py:118-131).

It is what ``bench.py --impl reference`` times (process pool over independent
units) and what the oracle pins compare ``eko`` with.
"""

from __future__ import annotations

import glob
import importlib.machinery
import importlib.util
import math
import multiprocessing as mp
import os

import numpy as np

from .eko import KINDS, wdtw_table

_HERE = os.path.dirname(os.path.abspath(__file__))
_MODE = {"squared": 0, "absolute": 1}


def ref_path():
    hits = sorted(glob.glob(os.path.join(_HERE, "_ref", "_speedups*.so")))
    return hits[0] if hits else None


_SP = None


def speedups():
    """The reference's compiled ``_speedups`` module (built from its .pyx)."""
    global _SP
    if _SP is None:
        path = ref_path()
        if path is None:
            raise RuntimeError("oracle/_ref/_speedups*.so is not built (run `make -C oracle ref`)")
        loader = importlib.machinery.ExtensionFileLoader("_speedups", path)
        spec = importlib.util.spec_from_loader("_speedups", loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _SP = mod
    return _SP


def available() -> bool:
    try:
        speedups()
        return True
    except Exception:
        return False


def _pc(a, b, mode):
    if mode == "squared":
        d = a - b
        return d * d
    return abs(a - b)


def _erp_border(values, gap, mode, row):
    out = np.empty(len(values) + 1, dtype=np.float64)
    out[0] = 0.0
    acc = 0.0
    for k, v in enumerate(values, start=1):
        acc = acc + (_pc(v, gap, mode) if row else _pc(gap, v, mode))
        out[k] = acc
    return out


class Payload:
    """What make_recurrence hands the compiled kernel for one pair."""

    __slots__ = ("lines", "cols", "weights", "vb", "hb")

    def __init__(self, spec, s, t):
        s = np.ascontiguousarray(s, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        lines, cols = (s, t) if len(s) >= len(t) else (t, s)
        self.lines, self.cols = lines, cols
        empty = speedups().EMPTY
        self.weights = empty
        self.vb = self.hb = empty
        if spec.kind == "wdtw":
            self.weights = wdtw_table(float(spec.wdtw_g), max(len(lines), len(cols)))
        elif spec.kind == "erp":
            lv, cv = lines.tolist(), cols.tolist()
            self.vb = _erp_border(lv, spec.erp_gap, spec.cost_mode, True)
            self.hb = _erp_border(cv, spec.erp_gap, spec.cost_mode, False)


def _canonical_fn(spec, lv, cv, weights):
    mode = spec.cost_mode
    if spec.kind in ("dtw", "cdtw", "erp"):
        return lambda i, j: _pc(lv[i - 1], cv[j - 1], mode)
    if spec.kind == "wdtw":
        wt = weights.tolist()
        return lambda i, j: _pc(lv[i - 1], cv[j - 1], mode) * wt[abs(i - j)]
    if spec.kind == "msm":
        return lambda i, j: abs(lv[i - 1] - cv[j - 1])
    nu = spec.twe_nu

    def twe(i, j):
        sp = lv[i - 2] if i >= 2 else 0.0
        tp = cv[j - 2] if j >= 2 else 0.0
        dij = float(abs(i - j))
        return _pc(lv[i - 1], cv[j - 1], mode) + _pc(sp, tp, mode) + nu * (dij + dij)

    return twe


def _alt_row_fn(spec, lv, cv, canonical):
    mode = spec.cost_mode
    if spec.kind == "erp":
        return lambda i, j: _pc(lv[i - 1], spec.erp_gap, mode)
    if spec.kind == "msm":
        c = spec.msm_c

        def msm(i, j):
            x = lv[i - 2] if i >= 2 else lv[i - 1]
            y = cv[j - 1]
            npt = lv[i - 1]
            if x <= npt <= y or x >= npt >= y:
                return c
            d1, d2 = abs(npt - x), abs(npt - y)
            return c + (d1 if d1 < d2 else d2)

        return msm
    if spec.kind == "twe":
        nu, lam = spec.twe_nu, spec.twe_lambda
        return lambda i, j: _pc(lv[i - 1], lv[i - 2] if i >= 2 else 0.0, mode) + nu + lam
    return canonical


def diagonal_upper_bound(spec, p: Payload):
    lv, cv = p.lines.tolist(), p.cols.tolist()
    canonical = _canonical_fn(spec, lv, cv, p.weights)
    alt_row = _alt_row_fn(spec, lv, cv, canonical)
    nl, nc = len(lv), len(cv)
    total = 0.0
    for k in range(1, nc + 1):
        total += canonical(k, k)
    for i in range(nc + 1, nl + 1):
        total += alt_row(i, nc)
    return total


def _run(spec, p: Payload, engine, window, cutoff):
    return speedups().run(
        engine, p.lines, p.cols, KINDS.index(spec.kind), _MODE[spec.cost_mode], window, cutoff,
        spec.erp_gap or 0.0, spec.msm_c or 0.0, spec.twe_nu or 0.0, spec.twe_lambda or 0.0,
        p.weights, p.vb, p.hb,
    )


def distance(spec, variant, s, t, cutoff=math.inf):
    """engines.distance over the reference's compiled kernel -> (cost, cells)."""
    p = Payload(spec, s, t)
    nl, nc = len(p.lines), len(p.cols)
    window = spec.window if spec.window is not None else nl
    if variant == "base":
        if spec.window is None:
            return _run(spec, p, "base", 0, math.inf)
        return _run(spec, p, "ea", window, math.inf)
    if variant == "ea":
        return _run(spec, p, "ea", window, cutoff)
    if variant == "eapruned":
        return _run(spec, p, "eapruned", window, cutoff)
    if variant != "pruned_only":
        raise ValueError(variant)
    if window < nl - nc:
        return math.inf, 0
    return _run(spec, p, "eapruned", window, diagonal_upper_bound(spec, p))


def nn_search(spec, variant, query, candidates):
    """search.nn_search (lb="none") -> (d_nn, best, cells, computed, abandoned)."""
    d_nn, best, cells, comp, ab = math.inf, -1, 0, 0, 0
    for idx, cand in enumerate(candidates):
        cost, cc = distance(spec, variant, query, cand, cutoff=d_nn)
        cells += cc
        if math.isinf(cost):
            ab += 1
            continue
        comp += 1
        if cost < d_nn:
            d_nn, best = cost, idx
    return d_nn, best, cells, comp, ab


def znormalize(s):
    s = np.asarray(s, dtype=np.float64)
    mean = s.mean()
    std = s.std()
    if std < 1e-12:
        return np.zeros_like(s)
    return (s - mean) / std


def subsequence_search(spec, variant, query, reference, normalize, lo=0, hi=None):
    """search.subsequence_search (lb="none") over offsets [lo, hi) -> (offset, dist, cells)."""
    query = np.ascontiguousarray(query, dtype=np.float64)
    reference = np.ascontiguousarray(reference, dtype=np.float64)
    lq = len(query)
    if normalize:
        query = znormalize(query)
    hi = len(reference) - lq + 1 if hi is None else hi
    best_d, best_off, cells = math.inf, -1, 0
    for off in range(lo, hi):
        win = reference[off:off + lq]
        if normalize:
            win = znormalize(win)
        cost, cc = distance(spec, variant, query, win, cutoff=best_d)
        cells += cc
        if math.isinf(cost):
            continue
        if cost < best_d:
            best_d, best_off = cost, off
    return best_off, best_d, cells


# ---- process-pool sharding (processes, not threads) ----

_G = {}


def _nn_worker(qidx):
    g = _G
    d, b, cells, _, _ = nn_search(g["spec"], g["variant"], g["Q"][qidx], g["C"])
    return qidx, d, b, cells


def nn_pool(spec, variant, Q, Cands, procs=None):
    """nn_search for every query, queries sharded across a fork process pool."""
    procs = procs or len(os.sched_getaffinity(0))
    _G.update(spec=spec, variant=variant, Q=Q, C=list(Cands))
    nq = len(Q)
    idx = np.empty(nq, dtype=np.int64)
    dist = np.empty(nq, dtype=np.float64)
    cells = np.empty(nq, dtype=np.int64)
    if procs <= 1 or nq == 1:
        for q in range(nq):
            _, dist[q], idx[q], cells[q] = _nn_worker(q)
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            for q, d, b, cc in pool.imap_unordered(_nn_worker, range(nq)):
                dist[q], idx[q], cells[q] = d, b, cc
    return idx, dist, cells


def _pw_worker(i):
    g = _G
    X, spec, variant = g["X"], g["spec"], g["variant"]
    row = np.empty(len(X) - i - 1)
    cells = 0
    for k, j in enumerate(range(i + 1, len(X))):
        row[k], cc = distance(spec, variant, X[i], X[j])
        cells += cc
    return i, row, cells


def pairwise_pool(spec, X, variant="pruned_only", rows=None, procs=None):
    """Upper-triangle rows ``rows`` of the all-pairs matrix, rows sharded across processes."""
    procs = procs or len(os.sched_getaffinity(0))
    _G.update(spec=spec, variant=variant, X=[np.ascontiguousarray(x, dtype=np.float64) for x in X])
    rows = list(range(len(X))) if rows is None else list(rows)
    out, total = {}, 0
    if procs <= 1:
        for i in rows:
            _, out[i], cc = _pw_worker(i)
            total += cc
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            for i, row, cc in pool.imap_unordered(_pw_worker, rows):
                out[i] = row
                total += cc
    return out, total


def _ss_worker(span):
    g = _G
    lo, hi = span
    return subsequence_search(g["spec"], g["variant"], g["q"], g["ref"], g["normalize"], lo, hi)


def subsequence_pool(spec, variant, query, reference, normalize, lo=0, hi=None, chunk=4096, procs=None):
    """Offsets [lo, hi) in chunks across processes; merged by lexicographic (dist, offset)."""
    procs = procs or len(os.sched_getaffinity(0))
    hi = len(reference) - len(query) + 1 if hi is None else hi
    _G.update(spec=spec, variant=variant, q=query, ref=reference, normalize=normalize)
    spans = [(a, min(a + chunk, hi)) for a in range(lo, hi, chunk)]
    if procs <= 1:
        res = [_ss_worker(s) for s in spans]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_ss_worker, spans)
    best_off, best_d, cells = -1, math.inf, 0
    for o, d, cc in res:
        cells += cc
        if o >= 0 and (d < best_d or (d == best_d and o < best_off)):
            best_off, best_d = o, d
    return best_off, best_d, cells
