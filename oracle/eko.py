"""ctypes front end of the C oracle (``ek_oracle.c``) -- TEST INFRASTRUCTURE ONLY.

Specs are duck-typed: anything with the attributes of the reference
``DistanceSpec`` (pkg/src/elastik/kernels.py:26-67) works, so the reference's
own spec objects and the product's mirror can both be passed.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libek_oracle.so")

KINDS = ("dtw", "cdtw", "wdtw", "erp", "msm", "twe")
VARIANTS = ("base", "ea", "eapruned", "pruned_only")
ENGINES = ("base", "ea", "eapruned")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class _Spec(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("mode", C.c_int), ("variant", C.c_int),
        ("window", C.c_long),
        ("gap", C.c_double), ("msm_c", C.c_double), ("nu", C.c_double), ("lam", C.c_double),
        ("wtabs", C.POINTER(_dp)),
    ]


def build():
    """Compile libek_oracle.so (and oracle/_ref when the reference is present)."""
    subprocess.run(["make", "-s", "-C", _HERE, "all"], check=True)


@lru_cache(maxsize=1)
def lib():
    if not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE, "oracle"], check=True)
    L = C.CDLL(_LIB_PATH)
    L.eko_run.argtypes = [C.c_int, _dp, C.c_long, _dp, C.c_long, C.c_int, C.c_int, C.c_long,
                          C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                          _dp, _dp, _dp, _dp, _i64p]
    L.eko_distance.argtypes = [C.POINTER(_Spec), _dp, C.c_long, _dp, C.c_long, C.c_double, _dp, _i64p]
    L.eko_diag_ub.argtypes = [C.POINTER(_Spec), _dp, C.c_long, _dp, C.c_long]
    L.eko_diag_ub.restype = C.c_double
    L.eko_nn.argtypes = [C.POINTER(_Spec), _dp, _i64p, _i64p, C.c_long, _dp, _i64p, _i64p, C.c_long,
                         C.c_int, _i64p, _dp, _i64p, _i64p, _i64p]
    L.eko_pairwise.argtypes = [C.POINTER(_Spec), _dp, _i64p, _i64p, C.c_long, C.c_int, _dp, _i64p]
    L.eko_np_sum.argtypes = [_dp, C.c_long]
    L.eko_np_sum.restype = C.c_double
    L.eko_znormalize.argtypes = [_dp, C.c_long, _dp, _dp]
    L.eko_subseq.argtypes = [C.POINTER(_Spec), _dp, C.c_long, _dp, C.c_long, C.c_int, C.c_long,
                             C.c_int, _i64p, _dp, _i64p]
    return L


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_i64p)


def wdtw_weight(g: float, d: int, length: int) -> float:
    # kernels.py:80-82, same Python float arithmetic (math.exp from libm)
    return 1.0 / (1.0 + math.exp(-g * (d - length / 2.0)))


@lru_cache(maxsize=256)
def wdtw_table(g: float, length: int) -> np.ndarray:
    # kernels.py:85-92
    t = np.empty(length + 1, dtype=np.float64)
    for d in range(length + 1):
        t[d] = wdtw_weight(g, d, length)
    t.setflags(write=False)
    return t


class _SpecHolder:
    """Keeps the ctypes struct plus the arrays its pointers reference alive."""

    def __init__(self, spec, variant: str, lengths):
        if variant not in VARIANTS:
            raise ValueError(f"unknown variant {variant!r}")
        self.tables = {}
        self.ptrs = None
        wt = None
        if spec.kind == "wdtw":
            top = max(lengths) if lengths else 0
            self.ptrs = (_dp * (top + 1))()
            for m in set(int(x) for x in lengths):
                tab = wdtw_table(float(spec.wdtw_g), m)
                self.tables[m] = tab
                self.ptrs[m] = _d(tab)
            wt = C.cast(self.ptrs, C.POINTER(_dp))
        self.s = _Spec(
            KINDS.index(spec.kind), 0 if spec.cost_mode == "squared" else 1, VARIANTS.index(variant),
            -1 if spec.window is None else int(spec.window),
            float(spec.erp_gap or 0.0), float(spec.msm_c or 0.0),
            float(spec.twe_nu or 0.0), float(spec.twe_lambda or 0.0), wt,
        )


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def run(engine, lines, cols, kind, mode, window, cutoff, erp_gap, msm_c, twe_nu, twe_lambda,
        weights, vborder_vals, hborder_vals):
    """Same signature and meaning as the reference's ``_speedups.run``
    (pkg/src/elastik/_speedups.pyx:274-317); returns (cost, cells)."""
    lines, cols = _f64(lines), _f64(cols)
    w = _f64(weights) if len(weights) else None
    vb = _f64(vborder_vals) if len(vborder_vals) else None
    hb = _f64(hborder_vals) if len(hborder_vals) else None
    cost = C.c_double()
    cells = C.c_int64()
    rc = lib().eko_run(ENGINES.index(engine), _d(lines), len(lines), _d(cols), len(cols), kind, mode,
                       window, cutoff, erp_gap, msm_c, twe_nu, twe_lambda,
                       _d(w) if w is not None else None, _d(vb) if vb is not None else None,
                       _d(hb) if hb is not None else None, C.byref(cost), C.byref(cells))
    if rc:
        raise RuntimeError(f"eko_run failed ({rc})")
    return cost.value, cells.value


def distance(spec, variant, s, t, cutoff=math.inf):
    """engines.distance (engines.py:121-147) -> (cost, cells_computed)."""
    s, t = _f64(s), _f64(t)
    h = _SpecHolder(spec, variant, [max(len(s), len(t))])
    cost = C.c_double()
    cells = C.c_int64()
    rc = lib().eko_distance(C.byref(h.s), _d(s), len(s), _d(t), len(t), float(cutoff),
                            C.byref(cost), C.byref(cells))
    if rc:
        raise RuntimeError(f"eko_distance failed ({rc})")
    return cost.value, cells.value


def diagonal_upper_bound(spec, s, t):
    s, t = _f64(s), _f64(t)
    h = _SpecHolder(spec, "base", [max(len(s), len(t))])
    return lib().eko_diag_ub(C.byref(h.s), _d(s), len(s), _d(t), len(t))


def _ragged(series):
    if isinstance(series, np.ndarray) and series.ndim == 2:
        arr = _f64(series)
        n, L = arr.shape
        off = np.arange(n, dtype=np.int64) * L
        lens = np.full(n, L, dtype=np.int64)
        return arr.reshape(-1), off, lens
    parts = [_f64(x) for x in series]
    lens = np.array([len(p) for p in parts], dtype=np.int64)
    off = np.zeros(len(parts), dtype=np.int64)
    if len(parts) > 1:
        off[1:] = np.cumsum(lens)[:-1]
    flat = np.concatenate(parts) if parts else np.zeros(0)
    return _f64(flat), off, lens


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def nn(spec, variant, queries, candidates, threads=None):
    """Per query: the reference's serial nn_search scan (search.py:81-125, lb="none").

    Returns dict(nn_index, nn_distance, cells, computed, abandoned) of arrays.
    """
    Qf, qo, ql = _ragged(queries)
    Cf, co, cl = _ragged(candidates)
    nq, ncand = len(ql), len(cl)
    lens = [max(a, b) for a in set(ql.tolist()) for b in set(cl.tolist())]
    h = _SpecHolder(spec, variant, lens)
    idx = np.empty(nq, dtype=np.int64)
    dist = np.empty(nq, dtype=np.float64)
    cells = np.empty(nq, dtype=np.int64)
    comp = np.empty(nq, dtype=np.int64)
    ab = np.empty(nq, dtype=np.int64)
    rc = lib().eko_nn(C.byref(h.s), _d(Qf), _i(qo), _i(ql), nq, _d(Cf), _i(co), _i(cl), ncand,
                      int(threads or default_threads()), _i(idx), _d(dist), _i(cells), _i(comp), _i(ab))
    if rc:
        raise RuntimeError(f"eko_nn failed ({rc})")
    return dict(nn_index=idx, nn_distance=dist, cells=cells, computed=comp, abandoned=ab)


def pairwise(spec, X, variant="pruned_only", threads=None):
    """Full symmetric matrix of distance(spec, variant, X[i], X[j]); diagonal 0.0."""
    Xf, off, lens = _ragged(X)
    n = len(lens)
    h = _SpecHolder(spec, variant, lens.tolist())
    D = np.empty((n, n), dtype=np.float64)
    cells = np.empty(n, dtype=np.int64)
    rc = lib().eko_pairwise(C.byref(h.s), _d(Xf), _i(off), _i(lens), n,
                            int(threads or default_threads()), _d(D), _i(cells))
    if rc:
        raise RuntimeError(f"eko_pairwise failed ({rc})")
    return D, int(cells.sum())


def np_sum(a):
    a = _f64(a)
    return lib().eko_np_sum(_d(a), len(a))


def znormalize(s):
    s = _f64(s)
    out = np.empty_like(s)
    tmp = np.empty_like(s)
    if lib().eko_znormalize(_d(s), len(s), _d(out), _d(tmp)):
        raise ValueError("z-normalization needs at least 2 points")
    return out


def subsequence(spec, variant, query, reference, normalize, chunk=None, threads=None):
    """subsequence_search (search.py:163-215, lb="none") -> (offset, distance, cells).

    ``chunk=None`` runs the reference's single serial scan; a finite chunk runs
    independent scans per chunk of offsets (process-pool style) merged by the
    lexicographic (distance, offset) minimum -- the same answer.
    """
    q = _f64(query)
    ref = _f64(reference)
    if normalize:
        q = znormalize(q)
    nwin = len(ref) - len(q) + 1
    if nwin < 1:
        raise ValueError("query longer than reference")
    chunk = nwin if chunk is None else int(chunk)
    nch = (nwin + chunk - 1) // chunk
    h = _SpecHolder(spec, variant, [len(q)])
    bo = np.empty(nch, dtype=np.int64)
    bd = np.empty(nch, dtype=np.float64)
    cells = np.empty(nch, dtype=np.int64)
    rc = lib().eko_subseq(C.byref(h.s), _d(q), len(q), _d(ref), len(ref), int(bool(normalize)), chunk,
                          int(threads or default_threads()), _i(bo), _d(bd), _i(cells))
    if rc:
        raise RuntimeError(f"eko_subseq failed ({rc})")
    best_off, best_d = -1, math.inf
    for o, d in zip(bo.tolist(), bd.tolist()):
        if o >= 0 and (d < best_d or (d == best_d and o < best_off)):
            best_off, best_d = o, d
    return best_off, best_d, int(cells.sum())


def subsequence_profile(spec, query, reference, normalize, threads=None):
    """Per-offset distance(spec, "base", query, window) of every window (the
    search.py:189-213 loop with no running cutoff) -> float64 array."""
    q = _f64(query)
    ref = _f64(reference)
    if normalize:
        q = znormalize(q)
    nwin = len(ref) - len(q) + 1
    if nwin < 1:
        raise ValueError("query longer than reference")
    h = _SpecHolder(spec, "base", [len(q)])
    bo = np.empty(nwin, dtype=np.int64)
    bd = np.empty(nwin, dtype=np.float64)
    cells = np.empty(nwin, dtype=np.int64)
    rc = lib().eko_subseq(C.byref(h.s), _d(q), len(q), _d(ref), len(ref), int(bool(normalize)), 1,
                          int(threads or default_threads()), _i(bo), _d(bd), _i(cells))
    if rc:
        raise RuntimeError(f"eko_subseq failed ({rc})")
    return bd
