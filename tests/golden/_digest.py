"""Canonical digests of planner outputs, shared by make_golden.py (which runs
the reference) and the tests (which run the oracle port and the C++ planner)."""

from __future__ import annotations

import hashlib
import struct

import numpy as np

B200_BF16 = dict(name="b200-sm100a-bf16", num_cores=148, regs_per_core=65536, smem_per_core_bytes=232448,
                 global_bw_bytes_per_s=8_000_000_000_000, shared_bw_bytes_per_s=37_225_920_000_000,
                 peak_flops=1_649_800_000_000_000, default_active_blocks=1, active_blocks_per_core=1, align_elems=64)
B200_FFMA = dict(name="b200-sm100a-ffma", num_cores=148, regs_per_core=65536, smem_per_core_bytes=232448,
                 global_bw_bytes_per_s=8_000_000_000_000, shared_bw_bytes_per_s=37_225_920_000_000,
                 peak_flops=74_449_920_000_000, default_active_blocks=2, active_blocks_per_core=2, align_elems=32)
V100_LIKE = dict(name="v100-like", num_cores=80, regs_per_core=65536, smem_per_core_bytes=98304,
                 global_bw_bytes_per_s=900_000_000_000, shared_bw_bytes_per_s=15_700_000_000_000,
                 peak_flops=15_700_000_000_000, default_active_blocks=2, active_blocks_per_core=2, align_elems=8)
DESCRIPTORS = {"b200_bf16": B200_BF16, "b200_ffma": B200_FFMA, "v100_like": V100_LIKE}


def tcgen05_legal(space_axes, ext: dict, smem: dict) -> bool:
    """Python statement of the B200 legality extension (planner.cpp
    tcgen05_legal) used to monkeypatch the reference's enumerate_ukernels."""
    ai, aj = space_axes[-2], space_axes[-1]
    ti, tj, Ei, Ej = smem[ai], smem[aj], ext[ai], ext[aj]

    def lane_ok(t, E):
        return (t % 128 == 0 and t <= 256) or (t >= E and t <= 128)

    def col_ok(t, E):
        return t == 256 or (t >= E and t <= 256)

    if any(smem[a] % 64 for a in smem if a not in space_axes):
        return False
    return (lane_ok(ti, Ei) and col_ok(tj, Ej)) or (lane_ok(tj, Ej) and col_ok(ti, Ei))


def fhex(x: float) -> str:
    return struct.pack(">d", float(x)).hex()


def digest_candidates(tile_keys, retained, bundles) -> str:
    """tile_keys: [(reg tuple, smem tuple)], retained: [int],
    bundles: [(pad float, occ float, regs, saturated, cmr, kmem, blocks)]."""
    h = hashlib.sha256()
    for (r, s), st, b in zip(tile_keys, retained, bundles):
        h.update(repr((tuple(int(v) for v in r), tuple(int(v) for v in s), int(st))).encode())
        pad, occ, regs, sat, cmr, kmem, blocks = b
        h.update(repr((fhex(pad), fhex(occ), int(regs), bool(sat), fhex(cmr), fhex(kmem), int(blocks))).encode())
    return h.hexdigest()


def digest_pool(plan_keys) -> str:
    """plan_keys: [(nparts, ((tile_key, n), ...))]."""
    h = hashlib.sha256()
    for k in plan_keys:
        h.update(repr(k).encode())
    return h.hexdigest()


def plan_key(parts) -> tuple:
    """parts: [((reg tuple, smem tuple), n), ...] -> canonical plan key."""
    return (len(parts), tuple(((tuple(map(int, r)), tuple(map(int, s))), int(n)) for (r, s), n in parts))


def as_arrays(tile_keys):
    reg = np.array([r for r, _ in tile_keys], dtype=np.int64)
    smem = np.array([s for _, s in tile_keys], dtype=np.int64)
    return reg, smem
