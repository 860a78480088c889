"""Multi-GPU sharding of the batched entry points, one process per GPU.

Every unit of work is independent, so nothing on the data path is exchanged:

* 1-NN: the queries are split across ranks, each rank searches its shard against the
  full candidate set, and the per-query results are gathered.
* Subsequence search: the stride-1 windows are split into contiguous ranges; a rank
  reads its range plus the query length - 1 halo of the stream, and the ranks' best
  (distance, offset) records meet in one lexicographic minimum -- the same tie rule as
  on one GPU (lowest offset wins).
* All-pairs: the upper triangle (numpy.triu_indices order) is split into contiguous pair
  ranges; each rank computes its range in one call (the device maps pair indices to
  (i, j), search.pairwise_range), and the values are gathered and mirrored.

Each process computes on its own GPU: ``bind_device()`` (called by every helper when it
uses the library) selects ``LOCAL_RANK`` modulo the visible devices for torch and for the
library (``ek_init``), as torchrun launches one process per GPU.

The process group is torch.distributed's (NCCL between GPUs; gloo works for the
host-side logic).  ``compute`` hooks let tests run the sharding with another
backend of the same signature (the CPU oracle under gloo).
"""

from __future__ import annotations

import math
import os

import numpy as np

from . import search
from .kernels import DistanceSpec


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of n units for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


_BOUND = None


def bind_device(local_rank: int | None = None) -> int:
    """Bind this process to GPU ``LOCAL_RANK % device_count`` (torch current device and the
    library's context).  Returns the device index.  Idempotent."""
    global _BOUND
    from . import _lib

    if local_rank is None:
        local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n = _lib.lib().ek_device_count()
    if n <= 0:
        raise RuntimeError("no CUDA device for this rank (there is no CPU fallback)")
    dev = local_rank % n
    if _BOUND == dev:
        return dev
    try:
        import torch

        torch.cuda.set_device(dev)
    except ImportError:  # pragma: no cover - torch is the plumbing, not required by the library
        pass
    _lib.check(_lib.lib().ek_init(dev))
    _BOUND = dev
    return dev


def _group_info(group):
    import torch.distributed as dist

    return dist.get_rank(group), dist.get_world_size(group)


def _all_gather(obj, group):
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def nn_batch_sharded(spec: DistanceSpec, variant: str, queries, candidates, group=None, compute=None):
    """nn_batch over all ranks: returns the full (nn_index, nn_distance, cells, computed,
    abandoned) arrays on every rank, identical to a single-process nn_batch."""
    rank, world = _group_info(group)
    queries = list(queries) if not isinstance(queries, np.ndarray) else queries
    lo, hi = shard_range(len(queries), rank, world)
    if compute is None:
        bind_device()
    run = compute or search.nn_batch
    local = run(spec, variant, queries[lo:hi], candidates)
    parts = _all_gather(tuple(np.asarray(a) for a in local), group)
    return tuple(np.concatenate([p[k] for p in parts]) for k in range(len(parts[0])))


def subsequence_search_sharded(query, reference, cfg, group=None, compute=None):
    """subsequence_search over all ranks -> (offset, distance, stats) on every rank.

    Rank r searches the windows starting in its share of [0, n_ref - lq]; it reads the
    stream up to lq - 1 points past its last start (the halo).  A rank whose share is
    empty contributes (+inf, -1)."""
    rank, world = _group_info(group)
    reference = np.asarray(reference, dtype=np.float64)
    lq = len(query)
    nwin = len(reference) - lq + 1
    lo, hi = shard_range(max(nwin, 0), rank, world)
    best = (math.inf, -1, 0, 0, 0)
    if hi > lo:
        if compute is None:
            bind_device()
        run = compute or search.subsequence_search
        off, d, st = run(query, reference[lo:hi + lq - 1], cfg)
        best = (d, off + lo if off >= 0 else -1, st.computed, st.abandoned, st.cells)
    parts = _all_gather(best, group)
    d_best, o_best = math.inf, -1
    for d, o, *_ in parts:  # lexicographic (distance, offset) minimum
        if o >= 0 and (d < d_best or (d == d_best and o < o_best)):
            d_best, o_best = d, o
    stats = search.SearchStats(computed=sum(p[2] for p in parts), abandoned=sum(p[3] for p in parts),
                               cells=sum(p[4] for p in parts))
    return o_best, d_best, stats


def pairwise_sharded(spec: DistanceSpec, X, variant: str = "pruned_only", group=None, compute=None):
    """The symmetric all-pairs matrix over all ranks -> (D, cells) on every rank.

    Rank r computes the contiguous pair range shard_range(n(n-1)/2, r, world) of the upper
    triangle (numpy.triu_indices order) with one ``pairwise_range`` call; the ranges are
    gathered and mirrored (diagonal 0.0).  ``compute(spec, variant, X, lo, hi) -> (costs,
    cells)`` replaces the library (tests)."""
    rank, world = _group_info(group)
    X = [np.asarray(x, dtype=np.float64) for x in X]
    n = len(X)
    lo, hi = shard_range(n * (n - 1) // 2, rank, world)
    if compute is None:
        bind_device()
    run = compute or search.pairwise_range
    costs, cells = run(spec, X, lo, hi, variant) if compute is None else run(spec, variant, X, lo, hi)
    parts = _all_gather((lo, hi, np.asarray(costs), int(cells)), group)
    iu, ju = np.triu_indices(n, k=1)
    D = np.zeros((n, n), dtype=np.float64)
    total = 0
    for plo, phi, c, ce in parts:
        D[iu[plo:phi], ju[plo:phi]] = c
        D[ju[plo:phi], iu[plo:phi]] = c
        total += ce
    return D, total
