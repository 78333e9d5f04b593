"""Multi-GPU execution of many independent dynamic shapes.

Shapes are independent problems, so they are partitioned across ranks by
shape bucket with an LPT (longest-processing-time) assignment on their
roofline time; every rank plans and executes its own bucket with one
persistent launch. There is no collective on the data path: the only
communication is an OPTIONAL final gather of per-shape records (checksum,
plan, timing) to rank 0 — over NCCL on GPUs, gloo in the CPU tests.

Launch one process per GPU (torchrun); ranks read RANK / WORLD_SIZE.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import asdict, dataclass

from .workloads import Shape, shard_lpt


@dataclass
class ShapeRecord:
    index: int
    kind: str
    name: str
    batch: int
    M: int
    N: int
    K: int
    plan: dict
    tuning_s: float
    checksum: str | None = None


def plan_bucket(shapes: list[Shape], indices: list[int], planner) -> list[ShapeRecord]:
    """Plan this rank's bucket (C++ planner, host thread pool)."""
    mine = [shapes[i] for i in indices]
    recs = planner.plan([s.instance() for s in mine]) if mine else []
    out = []
    for i, s, r in zip(indices, mine, recs):
        out.append(ShapeRecord(i, s.kind, s.name, s.batch, s.M, s.N, s.K, r.describe(), r.tuning_s))
    return out


def plan_digest(rec: ShapeRecord) -> str:
    blob = json.dumps({"shape": [rec.kind, rec.batch, rec.M, rec.N, rec.K], "parts": rec.plan["parts"],
                       "tau": rec.plan["tau"]}, sort_keys=True)
    return hashlib.sha256(blob.encode()).hexdigest()[:16]


def gather_records(records: list[ShapeRecord], rank: int, world: int, dst: int = 0):
    """Optional final gather (torch.distributed object gather). Returns the
    merged, index-ordered list on ``dst`` and None elsewhere."""
    if world == 1:
        return sorted(records, key=lambda r: r.index)
    import torch.distributed as dist

    payload = [asdict(r) for r in records]
    box = [None] * world if rank == dst else None
    dist.gather_object(payload, box, dst=dst)
    if rank != dst:
        return None
    merged = [ShapeRecord(**d) for part in box for d in part]
    return sorted(merged, key=lambda r: r.index)


def run_sharded(shapes: list[Shape], rank: int, world: int, planner, peak_flops: float, execute=None):
    """Partition, plan (and optionally execute) this rank's bucket; gather to rank 0."""
    buckets = shard_lpt(shapes, world, peak_flops)
    recs = plan_bucket(shapes, buckets[rank], planner)
    if execute is not None:
        execute([shapes[r.index] for r in recs], recs)
    return buckets, gather_records(recs, rank, world)
