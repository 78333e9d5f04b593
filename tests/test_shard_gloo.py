"""Multi-rank shape sharding on CPU (gloo, world_size 2): the LPT partition
covers every shape exactly once, each rank plans its own bucket with the C++
planner, and the gathered records equal single-process planning."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2407_21418_b200.workloads import c4_shapes, shard_lpt

PEAK = 1.6498e15


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_21418_b200.runtime import Planner
        from paper_2407_21418_b200.shard import plan_digest, run_sharded

        shapes = c4_shapes(n, seed=3)
        buckets, merged = run_sharded(shapes, rank, world, Planner(threads=2), PEAK)
        if rank == 0:
            q.put({"buckets": buckets, "digests": [plan_digest(r) for r in merged],
                   "indices": [r.index for r in merged]})
    finally:
        dist.destroy_process_group()


def test_lpt_partition_balanced_and_complete():
    shapes = c4_shapes(400, seed=1)
    for world in (1, 2, 4, 8):
        b = shard_lpt(shapes, world, PEAK)
        flat = sorted(i for part in b for i in part)
        assert flat == list(range(len(shapes)))
        loads = [sum(shapes[i].t_roof(PEAK) for i in part) for part in b]
        assert max(loads) <= min(loads) + max(s.t_roof(PEAK) for s in shapes) + 1e-12


def test_gloo_two_ranks_match_single_process():
    n = 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2407_21418_b200.runtime import Planner
    from paper_2407_21418_b200.shard import plan_bucket, plan_digest

    shapes = c4_shapes(n, seed=3)
    single = plan_bucket(shapes, list(range(n)), Planner(threads=2))
    assert res["indices"] == list(range(n))
    assert res["digests"] == [plan_digest(r) for r in single]
    assert sorted(i for b in res["buckets"] for i in b) == list(range(n))
