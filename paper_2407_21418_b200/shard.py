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
    """Partition, plan (and optionally execute) this rank's bucket; gather to
    rank 0. ``execute(shapes, records)`` runs the bucket and fills each
    record's ``checksum`` (a JSON string); the records — plan, tuning
    seconds, checksum — are the only thing that crosses ranks."""
    buckets = shard_lpt(shapes, world, peak_flops)
    recs = plan_bucket(shapes, buckets[rank], planner)
    if execute is not None:
        execute([shapes[r.index] for r in recs], recs)
    return buckets, gather_records(recs, rank, world)


def checksum_ok(cs: dict, rel: float = 1e-3) -> bool:
    """A shape's output checksum against its size-independent expectation
    (sum C == 1^T A B 1), relative to sum |C|."""
    return abs(cs["sum"] - cs["expect"]) <= rel * (cs["abs"] + 1.0)


def make_gpu_executor(planner, device, max_chunk_bytes: float = 12e9, time_launches: bool = True):
    """An ``execute`` for run_sharded on one GPU: the bucket runs in chunks of
    shapes whose operands + outputs fit ``max_chunk_bytes``; each chunk is ONE
    grouped launch of its lowered table (timed with CUDA events after one
    untimed launch), inputs seeded per GLOBAL shape index (so checksums do not
    depend on the partition). Fills record.checksum and returns a stats dict
    (kernel ms, launches, tables) through ``executor.stats``."""
    import json as _json

    import torch

    from .shapeset import ShapeSet

    stats = {"kernel_ms": 0.0, "launches": 0, "chunks": 0, "true_flops": 0, "t_roof_s": 0.0}

    def execute(shapes: list[Shape], records: list[ShapeRecord]):
        recs = planner.plan([s.instance() for s in shapes]) if shapes else []  # cache hits
        i = 0
        while i < len(shapes):
            j, size = i, 0.0
            while j < len(shapes) and (j == i or size + shapes[j].bytes_padded <= max_chunk_bytes):
                size += shapes[j].bytes_padded
                j += 1
            ss = ShapeSet(shapes[i:j], planner, device=device, seeds=[1000 * 4 + r.index for r in records[i:j]],
                          records=recs[i:j])
            s = torch.cuda.current_stream(device)
            ss.launch(s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ss.launch(s)
            e1.record(s)
            torch.cuda.synchronize(device)
            if time_launches:
                stats["kernel_ms"] += e0.elapsed_time(e1)
            stats["launches"] += 2
            stats["chunks"] += 1
            for rec, cs in zip(records[i:j], ss.checksums()):
                rec.checksum = _json.dumps(cs, sort_keys=True)
            del ss
            i = j
        stats["true_flops"] += sum(x.flops for x in shapes)

    execute.stats = stats
    return execute
