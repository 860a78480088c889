"""World-size-2 coverage of the multi-GPU sharding logic (gloo, CPU).

bench.py shards independent units across ranks with no data-path collective:
each rank searches its own query set (shard_seed) against the same candidates,
and only one scalar (the step time) is max-reduced.  Here two gloo ranks run the
CPU oracle on their shards; the union must equal a single-process run of the
same queries, and dist_max must return the max over ranks.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import bench
    from oracle import eko
    from paper_2102_05221_b200 import DistanceSpec, datagen

    r, w = bench.dist_init("gloo")
    assert (r, w) == (rank, world)
    C, _, protos = datagen.warped_prototypes(64, 48, 4, 0.1, 11)
    Q, _, _ = datagen.warped_prototypes(6, 48, 4, 0.1, bench.shard_seed(11, rank), protos=protos)
    res = eko.nn(DistanceSpec(kind="cdtw", window=5), "eapruned", Q, C, threads=1)
    t = bench.dist_max(float(rank + 1))
    bench.dist_barrier()
    gathered = [None] * world
    dist.all_gather_object(gathered, (Q, res["nn_index"], res["nn_distance"]))
    if rank == 0:
        out.put((t, gathered))
    dist.destroy_process_group()
    _ = torch


@pytest.mark.timeout(300)
def test_two_rank_query_shards_match_serial():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    t, gathered = out.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0  # max over ranks
    from oracle import eko
    from paper_2102_05221_b200 import DistanceSpec, datagen

    C, _, _ = datagen.warped_prototypes(64, 48, 4, 0.1, 11)
    Qs = np.concatenate([g[0] for g in gathered])
    assert not np.array_equal(gathered[0][0], gathered[1][0])  # distinct shards
    ref = eko.nn(DistanceSpec(kind="cdtw", window=5), "eapruned", Qs, C, threads=2)
    assert np.array_equal(np.concatenate([g[1] for g in gathered]), ref["nn_index"])
    assert np.array_equal(np.concatenate([g[2] for g in gathered]), ref["nn_distance"])


def _oracle_hooks():
    """CPU stand-ins with the signatures of nn_batch / subsequence_search / distance_batch."""
    from oracle import eko
    from paper_2102_05221_b200.search import SearchStats

    def nn(spec, variant, Q, C):
        r = eko.nn(spec, variant, Q, C, threads=1)
        return r["nn_index"], r["nn_distance"], r["cells"], r["computed"], r["abandoned"]

    def subseq(q, ref, cfg):
        off, d, cells = eko.subsequence(cfg.spec, cfg.variant, q, ref, cfg.normalize, threads=1)
        return off, d, SearchStats(cells=cells)

    def pairs(spec, variant, X, lo, hi):  # pairs [lo, hi) in np.triu_indices order
        iu, ju = np.triu_indices(len(X), k=1)
        out = [eko.distance(spec, variant, X[iu[k]], X[ju[k]]) for k in range(lo, hi)]
        return np.array([o[0] for o in out]), int(sum(o[1] for o in out))

    return nn, subseq, pairs


def _sharded_worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2102_05221_b200 import DistanceSpec, SearchConfig, datagen, distributed

    dist.init_process_group("gloo", rank=rank, world_size=world)
    nn, subseq, pairs = _oracle_hooks()
    C, _, protos = datagen.warped_prototypes(40, 40, 4, 0.1, 21)
    Q, _, _ = datagen.warped_prototypes(7, 40, 4, 0.1, 22, protos=protos)
    spec = DistanceSpec(kind="cdtw", window=4)
    res_nn = distributed.nn_batch_sharded(spec, "eapruned", Q, C, compute=nn)
    rng = np.random.default_rng(5)
    stream = np.cumsum(rng.normal(0, 1, 700))
    q = stream[311:351].copy()
    cfg = SearchConfig(spec=spec, variant="eapruned", normalize=True)
    res_ss = distributed.subsequence_search_sharded(q, stream, cfg, compute=subseq)
    X = [np.cumsum(rng.normal(0, 1, 25)) for _ in range(9)]
    res_pw = distributed.pairwise_sharded(DistanceSpec(kind="erp", window=5, erp_gap=0.0), X, compute=pairs)
    if rank == 0:
        out.put((res_nn, res_ss[:2], res_pw))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharded_entry_points_match_single_process():
    """distributed.{nn_batch,subsequence_search,pairwise}_sharded over 2 gloo ranks give the
    single-process answers (the stream split keeps its L-1 halo and the tie rule)."""
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    res_nn, res_ss, res_pw = out.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import eko
    from paper_2102_05221_b200 import DistanceSpec, datagen, distributed

    C, _, protos = datagen.warped_prototypes(40, 40, 4, 0.1, 21)
    Q, _, _ = datagen.warped_prototypes(7, 40, 4, 0.1, 22, protos=protos)
    spec = DistanceSpec(kind="cdtw", window=4)
    ref = eko.nn(spec, "eapruned", Q, C, threads=2)
    assert np.array_equal(res_nn[0], ref["nn_index"]) and np.array_equal(res_nn[1], ref["nn_distance"])
    rng = np.random.default_rng(5)
    stream = np.cumsum(rng.normal(0, 1, 700))
    q = stream[311:351].copy()
    off, d, _ = eko.subsequence(spec, "eapruned", q, stream, True)
    assert tuple(res_ss) == (off, d) and off == 311
    X = [np.cumsum(rng.normal(0, 1, 25)) for _ in range(9)]
    D = eko.pairwise(DistanceSpec(kind="erp", window=5, erp_gap=0.0), X)[0]
    assert np.array_equal(res_pw[0], D)
    assert [distributed.shard_range(7, r, 3) for r in range(3)] == [(0, 3), (3, 5), (5, 7)]


def _gpu_sharded_worker(rank, world, port, out):
    """Both ranks call the REAL library (bind_device: LOCAL_RANK % device count -> both on
    cuda:0 of a one-GPU box; their kernels never wait on each other)."""
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2102_05221_b200 import DistanceSpec, SearchConfig, datagen, distributed

    dist.init_process_group("gloo", rank=rank, world_size=world)
    C, _, protos = datagen.warped_prototypes(300, 128, 4, 0.1, 61)
    Q, _, _ = datagen.warped_prototypes(21, 128, 4, 0.1, 62, protos=protos)
    res_nn = distributed.nn_batch_sharded(DistanceSpec(kind="cdtw", window=12), "eapruned", Q, C)
    rng = np.random.default_rng(7)
    stream = np.cumsum(rng.normal(0, 1, 5000))
    q = stream[2711:2811].copy()
    cfg = SearchConfig(spec=DistanceSpec(kind="cdtw", window=5), variant="eapruned", normalize=True)
    res_ss = distributed.subsequence_search_sharded(q, stream, cfg)
    X = datagen.warped_prototypes(61, 96, 3, 0.1, 63)[0]
    res_pw = {k: distributed.pairwise_sharded(spec, X)[0] for k, spec in
              (("erp", DistanceSpec(kind="erp", window=9, erp_gap=0.0)), ("wdtw", DistanceSpec(kind="wdtw", wdtw_g=0.05)),
               ("msm", DistanceSpec(kind="msm", msm_c=0.5)))}
    if rank == 0:
        out.put((res_nn[:2], res_ss[:2], res_pw, distributed._BOUND))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_rank_sharded_on_the_gpu_library_match_single_process(gpu):
    """distributed.* over 2 gloo ranks on the real CUDA library equal one process's answers
    (bit for bit), including the subsequence halo and the all-pairs pair ranges."""
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_sharded_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    res_nn, res_ss, res_pw, bound = out.get(timeout=500)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert bound == 0
    from paper_2102_05221_b200 import DistanceSpec, SearchConfig, datagen

    C, _, protos = datagen.warped_prototypes(300, 128, 4, 0.1, 61)
    Q, _, _ = datagen.warped_prototypes(21, 128, 4, 0.1, 62, protos=protos)
    idx, dist_ = gpu.nn_batch(DistanceSpec(kind="cdtw", window=12), "eapruned", Q, C)[:2]
    assert np.array_equal(res_nn[0], idx) and np.array_equal(res_nn[1], dist_)
    rng = np.random.default_rng(7)
    stream = np.cumsum(rng.normal(0, 1, 5000))
    q = stream[2711:2811].copy()
    cfg = SearchConfig(spec=DistanceSpec(kind="cdtw", window=5), variant="eapruned", normalize=True)
    assert tuple(res_ss) == tuple(gpu.subsequence_search(q, stream, cfg)[:2]) and res_ss[0] == 2711
    X = datagen.warped_prototypes(61, 96, 3, 0.1, 63)[0]
    for k, spec in (("erp", DistanceSpec(kind="erp", window=9, erp_gap=0.0)), ("wdtw", DistanceSpec(kind="wdtw", wdtw_g=0.05)),
                    ("msm", DistanceSpec(kind="msm", msm_c=0.5))):
        assert np.array_equal(res_pw[k], gpu.pairwise(spec, X)[0]), k
