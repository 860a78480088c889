"""ctypes binding of the C ABI (include/elastik_b200.h) -> libelastik_b200.so.

There is no CPU fallback: if the library is missing or no CUDA device is
present, every call raises ``RuntimeError``.  Calls release the GIL (ctypes).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from functools import lru_cache

import numpy as np

from .errors import SpecError
from .kernels import KINDS, DistanceSpec, wdtw_weight_table

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libelastik_b200.so")

VARIANT_CODE = {"base": 0, "ea": 1, "eapruned": 2, "pruned_only": 3}

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class EkSpec(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("cost_mode", C.c_int32), ("window", C.c_int64),
        ("erp_gap", C.c_double), ("msm_c", C.c_double), ("twe_nu", C.c_double), ("twe_lambda", C.c_double),
        ("wdtw_tables", _dp), ("wdtw_table_off", _i64p), ("wdtw_max_len", C.c_int64),
        ("precision", C.c_int32),
    ]


PRECISIONS = ("float64", "float32")


def precision_code(precision: str) -> int:
    """``float64`` (default): the reference's arithmetic, bit-identical results.
    ``float32``: the optional faster mode (values within 1e-5 relative; not part of
    the reference's API)."""
    if precision not in PRECISIONS:
        raise SpecError(f"unknown precision {precision!r}; expected one of {PRECISIONS}")
    return PRECISIONS.index(precision)


EXPORTS = {
    "ek_last_error": ([], C.c_char_p),
    "ek_version": ([], C.c_char_p),
    "ek_device_count": ([], C.c_int),
    "ek_init": ([C.c_int], C.c_int),
    "ek_launch_count": ([C.c_int32], C.c_int64),
    "ek_set_profiling": ([C.c_int32], None),
    "ek_phase_times": ([_dp, C.POINTER(C.c_char_p), C.c_int32], C.c_int32),
    "ek_fp64_peak_ops": ([], C.c_double),
    "ek_fp32_peak_ops": ([], C.c_double),
    "ek_distance_batch": ([C.POINTER(EkSpec), C.c_int32, C.c_int64, _dp, C.c_int64, _i64p, _i64p, _i64p, _i64p,
                           _dp, _i64p, _dp, _i64p], C.c_int),
    "ek_run_batch": ([C.POINTER(EkSpec), C.c_int32, C.c_int64, _dp, C.c_int64, _i64p, _i64p, _i64p, _i64p,
                      _i64p, _dp, _dp, _i64p], C.c_int),
    "ek_nn": ([C.POINTER(EkSpec), C.c_int32, _dp, C.c_int64, _i64p, _i64p, C.c_int64, _dp, C.c_int64, _i64p, _i64p,
               C.c_int64, _i64p, _dp, _i64p, _i64p, _i64p], C.c_int),
    "ek_nn_submit": ([C.POINTER(EkSpec), C.c_int32, _dp, C.c_int64, _i64p, _i64p, C.c_int64, _dp, C.c_int64, _i64p,
                      _i64p, C.c_int64, C.c_int32], C.c_int),
    "ek_nn_collect": ([C.c_int32, _i64p, _dp, _i64p, _i64p, _i64p], C.c_int),
    "ek_nn_dev": ([C.POINTER(EkSpec), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                   C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                   C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "ek_pairwise": ([C.POINTER(EkSpec), C.c_int32, _dp, C.c_int64, _i64p, _i64p, C.c_int64, _dp, _i64p], C.c_int),
    "ek_pairwise_range": ([C.POINTER(EkSpec), C.c_int32, _dp, C.c_int64, _i64p, _i64p, C.c_int64, C.c_int64, C.c_int64,
                           _dp, _i64p], C.c_int),
    "ek_pairwise_dev": ([C.POINTER(EkSpec), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                         C.c_int32, C.c_void_p, _i64p, C.c_void_p], C.c_int),
    "ek_subseq": ([C.POINTER(EkSpec), C.c_int32, _dp, C.c_int64, _dp, C.c_int64, C.c_int32, _i64p, _dp, _i64p,
                   _i64p, _i64p], C.c_int),
    "ek_subseq_dev": ([C.POINTER(EkSpec), C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                       _i64p, _dp, _i64p, _i64p, _i64p, C.c_void_p], C.c_int),
    "ek_subseq_profile": ([C.POINTER(EkSpec), _dp, C.c_int64, _dp, C.c_int64, C.c_int32, _dp], C.c_int),
    "ek_envelopes": ([_dp, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int64, _dp, _dp], C.c_int),
    "ek_parse_tsv": ([C.c_char_p, C.c_int64, C.c_int32, _i64p, _i64p, _i64p, _i64p, _i64p, _dp, _i64p], C.c_int),
    "ek_host_alloc": ([C.c_int64], C.c_void_p),
    "ek_host_free": ([C.c_void_p], C.c_int),
    "ek_dev_alloc": ([C.c_int64], C.c_void_p),
    "ek_dev_free": ([C.c_void_p], C.c_int),
    "ek_memcpy": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p], C.c_int),
    "ek_derivative_dev": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p],
                          C.c_int),
    "ek_znormalize_dev": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                           C.c_void_p], C.c_int),
}

_lock = threading.Lock()


@lru_cache(maxsize=1)
def lib():
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, (args, res) in EXPORTS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().ek_last_error().decode("utf-8", "replace")
        if msg == "time series values must all be finite":  # the library's input validation (as_series)
            raise ValueError(msg)
        raise RuntimeError(f"elastik_b200: {msg}")


def available() -> bool:
    """True when the library loads and a CUDA device is present."""
    try:
        return lib().ek_device_count() > 0
    except (OSError, RuntimeError):
        return False


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


class SpecHandle:
    """ek_spec plus the host arrays its pointers reference (WDTW tables)."""

    def __init__(self, spec: DistanceSpec, longest_lengths=(), window_override=None, precision="float64"):
        if spec.kind not in KINDS:
            raise SpecError(f"unknown distance kind {spec.kind!r}")
        self._keep = []
        tabs = offs = None
        mx = 0
        if spec.kind == "wdtw":
            lens = sorted(set(int(m) for m in longest_lengths))
            mx = lens[-1] if lens else 0
            offs = np.full(mx + 1, -1, dtype=np.int64)
            parts, pos = [], 0
            for m in lens:
                t = wdtw_weight_table(float(spec.wdtw_g), m)
                offs[m] = pos
                parts.append(t)
                pos += m + 1
            tabs = np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(1))
            self._keep += [tabs, offs]
        window = spec.window if window_override is None else window_override
        self.s = EkSpec(
            KINDS.index(spec.kind), 0 if spec.cost_mode == "squared" else 1,
            -1 if window is None else int(window),
            float(spec.erp_gap or 0.0), float(spec.msm_c or 0.0),
            float(spec.twe_nu or 0.0), float(spec.twe_lambda or 0.0),
            dptr(tabs) if tabs is not None else None, iptr(offs) if offs is not None else None, mx,
            precision_code(precision),
        )

    @property
    def ref(self):
        return C.byref(self.s)


def ragged(series_list):
    """Concatenate series -> (flat float64, offsets int64, lengths int64)."""
    lens = np.fromiter((len(x) for x in series_list), dtype=np.int64, count=len(series_list))
    off = np.zeros(len(series_list), dtype=np.int64)
    if len(series_list) > 1:
        np.cumsum(lens[:-1], out=off[1:])
    flat = np.ascontiguousarray(np.concatenate(series_list) if len(series_list) else np.zeros(0))
    return flat, off, lens
