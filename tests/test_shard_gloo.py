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


def _small_mixed_shapes(n, seed):
    """C4-like mix (Dense of the BERT/LLM N,K pairs and attention BMMs) at
    sizes the numpy stand-in executes in milliseconds."""
    import random

    from paper_2407_21418_b200.workloads import Shape

    rng = random.Random(seed)
    out = []
    for _ in range(n):
        if rng.random() < 0.5:
            N, K = rng.choice([(768, 768), (2304, 768), (768, 3072)])
            out.append(Shape("dense", "dense", 1, rng.randint(1, 64), N, K, "nk"))
        else:
            T = rng.randint(1, 40)
            if rng.random() < 0.5:
                out.append(Shape("bmm", "scores", 12, T, T, 64, "nk", ("i", "j")))
            else:
                out.append(Shape("bmm", "context", 12, T, 64, T, "kn", ("i", "k")))
    return out


def _cpu_execute(shapes, records):
    """CPU stand-in for make_gpu_executor: the oracle's numpy execution with
    inputs seeded by the GLOBAL shape index; fills record.checksum."""
    import json

    import numpy as np

    from oracle.execute_np import execute_dense_fp32

    for s, r in zip(shapes, records):
        rng = np.random.default_rng(4000 + r.index)
        A = rng.uniform(-1, 1, (s.batch, s.M, s.K)).astype(np.float32)
        B = rng.uniform(-1, 1, (s.batch, s.K, s.N)).astype(np.float32)
        C = execute_dense_fp32(A, B).astype(np.float64)
        expect = float((A.astype(np.float64).sum(-2) * B.astype(np.float64).sum(-1)).sum())
        r.checksum = json.dumps({"sum": float(C.sum()), "expect": expect, "abs": float(np.abs(C).sum())},
                                sort_keys=True)


def _exec_worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2407_21418_b200.runtime import Planner
        from paper_2407_21418_b200.shard import run_sharded

        shapes = _small_mixed_shapes(n, seed=7)
        buckets, merged = run_sharded(shapes, rank, world, Planner(threads=2), PEAK, execute=_cpu_execute)
        if rank == 0:
            q.put({"buckets": buckets, "indices": [r.index for r in merged],
                   "checksums": [r.checksum for r in merged]})
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_execute_and_gather_checksums():
    """run_sharded with an executor: each rank executes only its LPT bucket
    (numpy stand-in for the GPU executor), fills per-shape output checksums,
    and rank 0's gather holds every shape once, in index order, with the
    checksums a single process computes — each verified against its
    size-independent expectation sum(C) = 1^T A B 1."""
    import json

    from paper_2407_21418_b200.runtime import Planner
    from paper_2407_21418_b200.shard import checksum_ok, plan_bucket

    n = 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exec_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res["indices"] == list(range(n))
    assert all(len(b) > 0 for b in res["buckets"])
    shapes = _small_mixed_shapes(n, seed=7)
    single = plan_bucket(shapes, list(range(n)), Planner(threads=2))
    _cpu_execute(shapes, single)
    assert res["checksums"] == [r.checksum for r in single]
    assert all(checksum_ok(json.loads(c)) for c in res["checksums"])
