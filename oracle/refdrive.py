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
from collections import deque

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


def nn_search(spec, variant, query, candidates, lb="none", envelopes=None):
    """search.nn_search (search.py:81-125) -> (d_nn, best, cells, computed, abandoned, lb_skips).

    ``lb`` = "none" / "keogh" / "keogh2" with the reference's own LB tests (restated below);
    ``envelopes``: the candidates' envelopes (search._candidate_envelopes, built once per
    classify_1nn call)."""
    d_nn, best, cells, comp, ab, skips = math.inf, -1, 0, 0, 0, 0
    env_q = None
    if lb == "keogh2":
        env_q = build_envelope(query, spec.window if spec.window is not None else len(query))
    for idx, cand in enumerate(candidates):
        if envelopes is not None and len(cand) == len(query):
            if lb == "keogh":
                bound = lb_keogh(query, envelopes[idx], spec.cost_mode)
            else:
                bound = lb_keogh2(query, cand, envelopes[idx], env_q, d_nn, spec.cost_mode)
            if bound >= d_nn:
                skips += 1
                continue
        cost, cc = distance(spec, variant, query, cand, cutoff=d_nn)
        cells += cc
        if math.isinf(cost):
            ab += 1
            continue
        comp += 1
        if cost < d_nn:
            d_nn, best = cost, idx
    return d_nn, best, cells, comp, ab, skips


# ---- lower_bounds.py restated (pkg/src/elastik/lower_bounds.py:23-98): the reference's
# pure-Python envelope (monotone deques) and LB_Keogh / LB_Keogh2 tests

def build_envelope(s, window):
    """lower_bounds.build_envelope (:23-57) -> (upper, lower) lists."""
    values = np.asarray(s, dtype=np.float64).tolist()
    n = len(values)
    upper, lower = [0.0] * n, [0.0] * n
    maxq, minq = deque(), deque()
    right = 0
    for i in range(n):
        hi = min(n - 1, i + window)
        while right <= hi:
            v = values[right]
            while maxq and values[maxq[-1]] <= v:
                maxq.pop()
            maxq.append(right)
            while minq and values[minq[-1]] >= v:
                minq.pop()
            minq.append(right)
            right += 1
        lo = i - window
        while maxq[0] < lo:
            maxq.popleft()
        while minq[0] < lo:
            minq.popleft()
        upper[i] = values[maxq[0]]
        lower[i] = values[minq[0]]
    return upper, lower


def lb_keogh(q, env, cost_mode="squared"):
    """lower_bounds.lb_keogh (:60-85): left-to-right sum of the distances to the envelope."""
    upper, lower = env
    squared = cost_mode == "squared"
    total = 0.0
    for qi, u, lo in zip(np.asarray(q, dtype=np.float64).tolist(), upper, lower):
        if qi > u:
            d = qi - u
        elif qi < lo:
            d = lo - qi
        else:
            continue
        total += d * d if squared else d
    return total


def lb_keogh2(q, c, env_c, env_q, cutoff=math.inf, cost_mode="squared"):
    """lower_bounds.lb_keogh2 (:88-98): both orders, the second skipped past the cutoff."""
    first = lb_keogh(q, env_c, cost_mode)
    if first > cutoff:
        return first
    second = lb_keogh(c, env_q, cost_mode)
    return second if second > first else first


def candidate_envelopes(spec, candidates, lb):
    """search._candidate_envelopes (search.py:69-78)."""
    if lb == "none" or spec.kind not in ("dtw", "cdtw"):
        return None
    return [build_envelope(c, spec.window if spec.window is not None else len(c)) for c in candidates]


def znormalize(s):
    s = np.asarray(s, dtype=np.float64)
    mean = s.mean()
    std = s.std()
    if std < 1e-12:
        return np.zeros_like(s)
    return (s - mean) / std


def subsequence_search(spec, variant, query, reference, normalize, lo=0, hi=None, lb="none"):
    """search.subsequence_search (search.py:163-215) over offsets [lo, hi) -> (offset, dist, cells)."""
    query = np.ascontiguousarray(query, dtype=np.float64)
    reference = np.ascontiguousarray(reference, dtype=np.float64)
    lq = len(query)
    if normalize:
        query = znormalize(query)
    w = spec.window if spec.window is not None else lq
    env_q = build_envelope(query, w) if lb != "none" else None
    hi = len(reference) - lq + 1 if hi is None else hi
    best_d, best_off, cells = math.inf, -1, 0
    for off in range(lo, hi):
        win = reference[off:off + lq]
        if normalize:
            win = znormalize(win)
        if env_q is not None:
            bound = lb_keogh(win, env_q, spec.cost_mode)
            if lb == "keogh2" and bound < best_d:
                bound = lb_keogh2(query, win, build_envelope(win, w), env_q, best_d, spec.cost_mode)
            if bound >= best_d:
                continue
        cost, cc = distance(spec, variant, query, win, cutoff=best_d)
        cells += cc
        if math.isinf(cost):
            continue
        if cost < best_d:
            best_d, best_off = cost, off
    return best_off, best_d, cells


# ---- process-pool sharding (processes, not threads) ----
#
# The pools are created once per workload, before the timed region (fork copies the
# workload into every worker), and warmed with one task, so a timed step measures the
# steady-state scan, not process start-up.

_G = {}


def _nn_worker(qidx):
    g = _G
    d, b, cells, _, _, _ = nn_search(g["spec"], g["variant"], g["Q"][qidx], g["C"], g["lb"], g["env"])
    return qidx, d, b, cells


def _pw_worker(i):
    g = _G
    X, spec, variant = g["X"], g["spec"], g["variant"]
    row = np.empty(len(X) - i - 1)
    cells = 0
    for k, j in enumerate(range(i + 1, len(X))):
        row[k], cc = distance(spec, variant, X[i], X[j])
        cells += cc
    return i, row, cells


def _ss_worker(span):
    g = _G
    lo, hi = span
    return subsequence_search(g["spec"], g["variant"], g["q"], g["ref"], g["normalize"], lo, hi, g["lb"])


class _Pool:
    def __init__(self, procs, **workload):
        self.procs = procs or len(os.sched_getaffinity(0))
        _G.clear()
        _G.update(workload)
        self.pool = mp.get_context("fork").Pool(self.procs) if self.procs > 1 else None

    def map(self, fn, items):
        if self.pool is None:
            return [fn(x) for x in items]
        return list(self.pool.imap_unordered(fn, items))

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class NNPool(_Pool):
    """nn_search per query, queries sharded across a persistent fork pool.

    ``env`` (lb != "none"): the candidates' envelopes, built by the caller the way
    classify_1nn does (once per call, serially, search.py:140)."""

    def __init__(self, spec, variant, Q, Cands, lb="none", env=None, procs=None):
        super().__init__(procs, spec=spec, variant=variant, Q=Q, C=list(Cands), lb=lb, env=env)
        self.nq = len(Q)

    def warm(self):
        self.map(_nn_worker, [0] * (self.procs or 1))

    def run(self, queries):
        queries = list(queries)
        idx = np.empty(len(queries), dtype=np.int64)
        dist = np.empty(len(queries), dtype=np.float64)
        cells = np.empty(len(queries), dtype=np.int64)
        pos = {q: k for k, q in enumerate(queries)}
        for q, d, b, cc in self.map(_nn_worker, queries):
            dist[pos[q]], idx[pos[q]], cells[pos[q]] = d, b, cc
        return idx, dist, cells


class PairwisePool(_Pool):
    def __init__(self, spec, X, variant="pruned_only", procs=None):
        super().__init__(procs, spec=spec, variant=variant, X=[np.ascontiguousarray(x, dtype=np.float64) for x in X])
        self.n = len(X)

    def warm(self):
        self.map(_pw_worker, [self.n - 2] * (self.procs or 1))

    def run(self, rows):
        out, total = {}, 0
        for i, row, cc in self.map(_pw_worker, list(rows)):
            out[i] = row
            total += cc
        return out, total


class SubseqPool(_Pool):
    def __init__(self, spec, variant, query, reference, normalize, lb="none", procs=None):
        super().__init__(procs, spec=spec, variant=variant, q=query, ref=reference, normalize=normalize, lb=lb)

    def warm(self):
        self.map(_ss_worker, [(0, 2)] * (self.procs or 1))

    def run(self, lo, hi, chunk=4096):
        spans = [(a, min(a + chunk, hi)) for a in range(lo, hi, chunk)]
        best_off, best_d, cells = -1, math.inf, 0
        for o, d, cc in self.map(_ss_worker, spans):
            cells += cc
            if o >= 0 and (d < best_d or (d == best_d and o < best_off)):
                best_off, best_d = o, d
        return best_off, best_d, cells


def nn_pool(spec, variant, Q, Cands, procs=None, lb="none"):
    """nn_search for every query (one-shot pool)."""
    env = candidate_envelopes(spec, Cands, lb)
    with NNPool(spec, variant, Q, Cands, lb, env, procs) as p:
        return p.run(range(len(Q)))


def pairwise_pool(spec, X, variant="pruned_only", rows=None, procs=None):
    """Upper-triangle rows ``rows`` of the all-pairs matrix (one-shot pool)."""
    with PairwisePool(spec, X, variant, procs) as p:
        return p.run(range(len(X)) if rows is None else rows)


def subsequence_pool(spec, variant, query, reference, normalize, lo=0, hi=None, chunk=4096, procs=None, lb="none"):
    """Offsets [lo, hi) in chunks across processes; merged by lexicographic (dist, offset)."""
    hi = len(reference) - len(query) + 1 if hi is None else hi
    with SubseqPool(spec, variant, query, reference, normalize, lb, procs) as p:
        return p.run(lo, hi, chunk)
