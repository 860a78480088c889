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
