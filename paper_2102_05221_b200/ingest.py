"""Ingestion: UCR text files into page-locked packed batches, resident
device batches, and the series transforms of ``series.py`` on the GPU.

* :func:`load_tsv_packed` reads a UCR-format file (``series.load_tsv``,
  pkg/src/elastik/series.py:61-86) with the library's native parser (``ek_parse_tsv``) into
  one flat float64 buffer in page-locked memory plus offsets, lengths and labels -- the
  layout every entry point takes, ready for an asynchronous upload.  Any file the fast path
  does not decide (an irregular token, a non-finite value, a line without a value, an empty
  file, non-ASCII text) is loaded by the reference-semantics loader, so accepted files and
  raised errors (``ParseError`` with its line and column, ``EmptyDatasetError``) are exactly
  ``load_tsv``'s.
* :class:`DeviceSeries` keeps a batch (equal or unequal lengths) resident in HBM, so
  repeated searches against the same candidates do not re-upload them.
  :meth:`DeviceSeries.derivative` / :meth:`DeviceSeries.znormalize` are ``series.derivative``
  (series.py:134-144) and ``series.znormalize`` (series.py:118-131) on the device,
  bit-identical to the reference's numpy; :func:`nn_batch_device` is ``nn_batch`` on
  resident batches.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _backend, _lib
from .errors import DegenerateInputError, SearchError, SpecError
from .kernels import DistanceSpec
from .series import LabeledDataset, _separator, as_series, load_tsv

__all__ = ["PackedDataset", "load_tsv_packed", "pack", "DeviceSeries", "nn_batch_device"]


class _Pinned:
    """Page-locked host buffer (ek_host_alloc) viewed as a numpy array; freed with the view."""

    def __init__(self, nbytes: int):
        self.ptr = _lib.lib().ek_host_alloc(max(8, int(nbytes)))
        if not self.ptr:
            _lib.check(-1)
        self.nbytes = int(nbytes)

    def array(self, dtype, count):
        buf = (C.c_char * max(8, self.nbytes)).from_address(self.ptr)
        buf._pinned_owner = self  # the view's base keeps the allocation alive
        return np.frombuffer(buf, dtype=dtype, count=count)

    def __del__(self):
        if getattr(self, "ptr", None):
            try:
                _lib.lib().ek_host_free(self.ptr)
            except Exception:  # interpreter shutdown
                pass
            self.ptr = None


def _host_buffer(count: int, pinned: bool) -> np.ndarray:
    if pinned:
        try:
            return _Pinned(8 * count).array(np.float64, count)
        except (OSError, RuntimeError):
            pass  # no device: ordinary memory (the layout is the same)
    return np.empty(count, dtype=np.float64)


@dataclass
class PackedDataset:
    """A labelled batch in the library's packed layout: series s is
    ``values[offsets[s] : offsets[s] + lengths[s]]``."""

    name: str
    labels: np.ndarray    # int64 [n] (object: Python ints beyond int64)
    values: np.ndarray    # float64, page-locked when a device is present
    offsets: np.ndarray   # int64 [n]
    lengths: np.ndarray   # int64 [n]

    def __len__(self):
        return len(self.labels)

    def series(self, s: int) -> np.ndarray:
        o = int(self.offsets[s])
        return self.values[o:o + int(self.lengths[s])]

    @property
    def pinned(self) -> bool:
        return hasattr(self.values.base, "_pinned_owner")

    def to_labeled(self) -> LabeledDataset:
        return LabeledDataset(name=self.name, entries=tuple((int(self.labels[s]), self.series(s).copy())
                                                            for s in range(len(self))))


def pack(series, labels=None, name: str = "batch", pinned: bool = True) -> PackedDataset:
    """Pack series (validated with as_series) into the layout of :class:`PackedDataset`."""
    arrs = [as_series(x) for x in series]
    lens = np.fromiter((len(a) for a in arrs), dtype=np.int64, count=len(arrs))
    off = np.zeros(len(arrs), dtype=np.int64)
    if len(arrs) > 1:
        np.cumsum(lens[:-1], out=off[1:])
    vals = _host_buffer(int(lens.sum()), pinned)
    for a, o in zip(arrs, off):
        vals[o:o + len(a)] = a
    if labels is None:
        lab = np.zeros(len(arrs), dtype=np.int64)
    else:
        try:
            lab = np.asarray(labels, dtype=np.int64)
        except OverflowError:  # int(label) beyond int64 stays a Python int, as in load_tsv
            lab = np.array(list(labels), dtype=object)
    return PackedDataset(name, lab, vals, off, lens)


def load_tsv_packed(path, delimiter: str = "tab", name: str | None = None, pinned: bool = True) -> PackedDataset:
    """``series.load_tsv`` into a :class:`PackedDataset` (see the module docstring)."""
    sep = _separator(delimiter)
    with open(path, "rb") as fh:
        data = fh.read()
    L = _lib.lib()
    ns, nv, bad = np.zeros(1, np.int64), np.zeros(1, np.int64), np.zeros(1, np.int64)
    nil = C.POINTER(C.c_int64)()
    rc = L.ek_parse_tsv(data, len(data), ord(sep), _lib.iptr(ns), _lib.iptr(nv), nil, nil, nil,
                        C.POINTER(C.c_double)(), _lib.iptr(bad))
    if rc == 0:
        n, m = int(ns[0]), int(nv[0])
        lab, off, lens = (np.empty(n, np.int64) for _ in range(3))
        vals = _host_buffer(m, pinned)
        rc = L.ek_parse_tsv(data, len(data), ord(sep), _lib.iptr(ns), _lib.iptr(nv), _lib.iptr(lab), _lib.iptr(off),
                            _lib.iptr(lens), _lib.dptr(vals), _lib.iptr(bad))
        if rc == 0:
            return PackedDataset(str(path) if name is None else name, lab, vals, off, lens)
    if rc < 0:
        _lib.check(rc)
    # the reference-semantics loader decides (accepts exactly what load_tsv accepts, raises
    # its ParseError / EmptyDatasetError otherwise)
    ds = load_tsv(path, delimiter=delimiter, name=name)
    return pack(ds.series, ds.labels, ds.name, pinned)


class DeviceSeries:
    """A batch of series resident on the device (values float64, offsets int64, lengths
    int32), uploaded once; free() (or the context manager) releases it."""

    def __init__(self, values_ptr: int, offsets_ptr: int, lengths_ptr: int, lengths: np.ndarray, total: int):
        self._v, self._o, self._l = values_ptr, offsets_ptr, lengths_ptr
        self.lengths = np.asarray(lengths, dtype=np.int64)
        self.total = int(total)

    # -- construction ---------------------------------------------------------------
    @classmethod
    def _alloc(cls, lengths: np.ndarray):
        L = _lib.lib()
        lengths = np.asarray(lengths, dtype=np.int64)
        total = int(lengths.sum())
        off = np.zeros(len(lengths), dtype=np.int64)
        if len(lengths) > 1:
            np.cumsum(lengths[:-1], out=off[1:])
        ptrs = [L.ek_dev_alloc(8 * max(1, total)), L.ek_dev_alloc(8 * max(1, len(lengths))),
                L.ek_dev_alloc(4 * max(1, len(lengths)))]
        if not all(ptrs):
            for p in ptrs:
                if p:
                    L.ek_dev_free(p)
            _lib.check(-1)
        ds = cls(ptrs[0], ptrs[1], ptrs[2], lengths, total)
        _copy(ds._o, off, 0)
        _copy(ds._l, lengths.astype(np.int32), 0)
        return ds

    @classmethod
    def upload(cls, batch) -> "DeviceSeries":
        """Upload a :class:`PackedDataset`, a 2-D float64 array or a list of series (each
        validated like as_series)."""
        _backend.resolve(None)
        if isinstance(batch, PackedDataset):
            vals, off, lens = batch.values, batch.offsets, batch.lengths
            if len(lens) and not np.isfinite(vals[:int(lens.sum())]).all():
                raise ValueError("time series values must all be finite")
            if np.any(lens < 1):
                raise ValueError("time series must contain at least one value")
            contiguous = len(lens) == 0 or (off[0] == 0 and np.array_equal(off[1:], np.cumsum(lens)[:-1]))
            if not contiguous:
                batch = pack([batch.series(s) for s in range(len(batch))], pinned=False)
                vals, lens = batch.values, batch.lengths
        elif isinstance(batch, np.ndarray) and batch.ndim == 2:
            arr = np.ascontiguousarray(batch, dtype=np.float64)
            if arr.shape[1] < 1 and arr.shape[0]:
                raise ValueError("time series must contain at least one value")
            if not np.isfinite(arr).all():
                raise ValueError("time series values must all be finite")
            vals, lens = arr.reshape(-1), np.full(arr.shape[0], arr.shape[1], dtype=np.int64)
        else:
            p = pack(batch, pinned=False)
            vals, lens = p.values, p.lengths
        ds = cls._alloc(lens)
        _copy(ds._v, np.ascontiguousarray(vals[:ds.total]), 0)
        return ds

    # -- transforms -----------------------------------------------------------------
    def derivative(self) -> "DeviceSeries":
        """series.derivative of every series (two points shorter), on the device."""
        if np.any(self.lengths < 3):
            raise DegenerateInputError("derivative transform needs at least 3 points")
        out = DeviceSeries._alloc(self.lengths - 2)
        _lib.check(_lib.lib().ek_derivative_dev(self._v, self._o, self._l, len(self), out._v, out._o, None))
        return out

    def znormalize(self) -> "DeviceSeries":
        """series.znormalize of every series (numpy's mean / std), on the device."""
        if np.any(self.lengths < 2):
            raise DegenerateInputError("z-normalization needs at least 2 points")
        out = DeviceSeries._alloc(self.lengths)
        hl = self.lengths.astype(np.int32)
        _lib.check(_lib.lib().ek_znormalize_dev(self._v, self._o, self._l, hl.ctypes.data, len(self), out._v,
                                                out._o, None))
        return out

    # -- access ---------------------------------------------------------------------
    def __len__(self):
        return len(self.lengths)

    @property
    def dense(self) -> bool:
        return len(self.lengths) > 0 and bool(np.all(self.lengths == self.lengths[0]))

    def to_host(self) -> list:
        flat = np.empty(max(1, self.total), dtype=np.float64)
        _copy(flat, self._v, 1, 8 * self.total)
        out, o = [], 0
        for m in self.lengths:
            out.append(flat[o:o + int(m)].copy())
            o += int(m)
        return out

    def free(self):
        if getattr(self, "_v", None):
            L = _lib.lib()
            for p in (self._v, self._o, self._l):
                L.ek_dev_free(p)
            self._v = self._o = self._l = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()

    def __del__(self):
        try:
            self.free()
        except Exception:  # interpreter shutdown
            pass


def _copy(dst, src, direction: int, nbytes: int | None = None):
    """ek_memcpy between a device pointer (int) and a numpy array (synchronous)."""
    if direction == 0:  # host array -> device
        nbytes = src.nbytes if nbytes is None else nbytes
        _lib.check(_lib.lib().ek_memcpy(dst, src.ctypes.data, nbytes, 0, None))
    else:               # device -> host array
        _lib.check(_lib.lib().ek_memcpy(dst.ctypes.data, src, nbytes, 1, None))


def nn_batch_device(spec: DistanceSpec, variant: str, queries: DeviceSeries, candidates: DeviceSeries,
                    precision: str = "float64"):
    """``nn_batch`` on resident batches (no upload): the same 1-NN answers and statistics."""
    from .search import VARIANTS

    _backend.resolve(None)
    _lib.precision_code(precision)
    if variant not in VARIANTS:
        raise SpecError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    if len(candidates) == 0:
        raise SearchError("candidate set is empty")
    nq = len(queries)
    out = [np.empty(nq, dtype=np.int64), np.empty(nq, dtype=np.float64)] + [np.empty(nq, dtype=np.int64)
                                                                             for _ in range(3)]
    if nq == 0:
        return tuple(out)
    ql, cl = queries.lengths, candidates.lengths
    longest = np.unique(np.maximum.outer(np.unique(ql), np.unique(cl))) if spec.kind == "wdtw" else ()
    h = _lib.SpecHandle(spec, longest_lengths=longest, precision=precision)
    L = _lib.lib()
    mx = int(max(ql.max(), cl.max()))
    dense = int(queries.dense and candidates.dense and ql[0] == cl[0])
    dout = L.ek_dev_alloc(8 * 5 * nq)
    if not dout:
        _lib.check(-1)
    try:
        p = [dout + 8 * nq * k for k in range(5)]
        _lib.check(L.ek_nn_dev(h.ref, _lib.VARIANT_CODE[variant], queries._v, queries._o, queries._l, nq,
                               candidates._v, candidates._o, candidates._l, len(candidates), mx, dense,
                               p[0], p[1], p[2], p[3], p[4], None))
        flat = np.empty(5 * nq, dtype=np.int64)
        _copy(flat, dout, 1, 8 * 5 * nq)
    finally:
        L.ek_dev_free(dout)
    out[0][:] = flat[:nq]
    out[1][:] = flat[nq:2 * nq].view(np.float64)
    for k in range(2, 5):
        out[k][:] = flat[k * nq:(k + 1) * nq]
    return tuple(out)
