"""ORACLE — test infrastructure only (tests/, smoke(), bench.py cpu_baseline
and --impl reference). Never on the product path.

CPU restatement of executing a ProgramPlan: the reference stops at the plan
(combine.py:30-55); its coverage semantics (timemodel.py:78-96,
combine.py:44-55) define what execution means: part q covers count_q tiles
of size smem_q[tau] along tau starting after the previous parts; every other
space axis is tiled uniformly from 0 (the last tile ragged, padding never
written). Walking that tile grid and accumulating A[tile] @ B[tile] in fp32
proves the plan covers C exactly once and gives the reference output.
"""

from __future__ import annotations

import numpy as np


def execute_dense_fp32(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """C = A @ B in fp32 (numpy/OpenBLAS sgemm); A [b,M,K] or [M,K], B [b,K,N] / [K,N]."""
    return np.matmul(A.astype(np.float32, copy=False), B.astype(np.float32, copy=False))


def plan_tiles(extents: dict, space_axes: list, tau: str, parts: list):
    """Yield per-axis (lo, hi) ranges of every uKernel rectangle of a plan.

    ``parts`` = [(smem_tile dict, count), ...]."""
    off = 0
    for tiles, count in parts:
        t = tiles[tau]
        for c in range(count):
            ranges = []
            for s in space_axes:
                if s == tau:
                    ranges.append([(off, off + t)])
                else:
                    e, ts = extents[s], tiles[s]
                    ranges.append([(o, min(e, o + ts)) for o in range(0, e, ts)])
            off += t
            idx = [0] * len(space_axes)
            while True:
                yield tuple(ranges[d][idx[d]] for d in range(len(space_axes)))
                d = len(space_axes) - 1
                while d >= 0:
                    idx[d] += 1
                    if idx[d] < len(ranges[d]):
                        break
                    idx[d] = 0
                    d -= 1
                if d < 0:
                    break


def execute_plan(A: np.ndarray, B: np.ndarray, extents: dict, space_axes: list, tau: str, parts: list,
                 dtype=np.float32) -> tuple[np.ndarray, np.ndarray]:
    """Tile-by-tile execution of a Dense (i, j) or BMM (b, i, j) plan.

    Returns (C, coverage) where coverage counts how often each output element
    was written (must be all ones)."""
    bmm = len(space_axes) == 3
    if not bmm:
        A, B = A[None], B[None]
    nb, M, _ = A.shape
    N = B.shape[2]
    C = np.zeros((nb, M, N), dtype=dtype)
    cov = np.zeros((nb, M, N), dtype=np.int32)
    for rect in plan_tiles(extents, space_axes, tau, parts):
        (b0, b1), (i0, i1), (j0, j1) = rect if bmm else ((0, 1),) + rect
        C[b0:b1, i0:i1, j0:j1] = np.matmul(A[b0:b1, i0:i1, :].astype(dtype), B[b0:b1, :, j0:j1].astype(dtype))
        cov[b0:b1, i0:i1, j0:j1] += 1
    if not bmm:
        return C[0], cov[0]
    return C, cov
