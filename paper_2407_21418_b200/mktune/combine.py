"""Runtime-stage composition (drop-in for mktune.combine, combine.py:1-194).

The main axis tau is the largest space axis; a program covers it exactly
with one tile size or two (n1*a + n2*b = H); the two parts agree on every
other tile. ``build_programs`` enumerates that pool in the C++ planner and
returns it in the reference's canonical order; ``plan_pool_size`` counts it
without materialising anything (pools reach 10^8 plans at B200 shapes).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from .. import _lib
from . import _native
from .errors import EmptyResultError, InputError, InternalError
from .timemodel import TimeEstimate
from .ukernel import UKernel
from .workload import WorkloadInstance

Combo = tuple[tuple[int, int], ...]


@dataclass
class ProgramPlan:
    parts: tuple  # ((UKernel, count),) or ((UKernel, count), (UKernel, count))
    shape: WorkloadInstance
    tau: str
    sia: float | None = None
    est: TimeEstimate | None = None

    @property
    def tau_coverage(self) -> int:
        return sum(k.smem_tile[self.tau] * n for k, n in self.parts)

    def covered_extents(self) -> dict:
        out = {}
        for s in self.shape.spec.space_axes:
            if s == self.tau:
                out[s] = self.tau_coverage
            else:
                t = self.parts[0][0].smem_tile[s]
                out[s] = -(-self.shape.extent(s) // t) * t
        return out


def select_main_axis(instance: WorkloadInstance) -> str:
    spec = instance.spec
    if not spec.space_axes:
        raise InputError("workload has no space axes", field="axes")
    top = max(instance.extent(s) for s in spec.space_axes)
    tied = [s for s in spec.space_axes if instance.extent(s) == top]
    dyn = [s for s in tied if spec.axis(s).is_dynamic]
    return min(dyn or tied)


def _pair_solutions(a: int, b: int, extent: int) -> Iterable[tuple[int, int]]:
    """(n1, n2 >= 1) with n1*a + n2*b == extent, walking the residue class of n2."""
    g = math.gcd(a, b)
    if extent % g:
        return
    a_, b_, h = a // g, b // g, extent // g
    n2 = 1 if a_ == 1 else ((h * pow(b_, -1, a_)) % a_ or a_)
    while n2 * b_ <= h - a_:
        yield (h - n2 * b_) // a_, n2
        n2 += a_


def combin_search(tile_sizes: Iterable[int], extent: int) -> set[Combo]:
    if extent < 1:
        raise InputError(f"extent must be >= 1, got {extent}")
    tiles = sorted({int(t) for t in tile_sizes})
    if not tiles or tiles[0] < 1:
        raise InputError("tile sizes must be positive integers")
    found: set[Combo] = {((t, extent // t),) for t in tiles if extent % t == 0}
    for x, a in enumerate(tiles):
        if a > extent:
            break
        for b in tiles[x + 1:]:
            found.update(((a, n1), (b, n2)) for n1, n2 in _pair_solutions(a, b, extent))
    return found


def _part_signature(k: UKernel, tau: str, space_axes: Sequence[str], axis_names: Sequence[str]) -> tuple:
    return (tuple(k.reg_tile[a] for a in space_axes if a != tau), tuple(k.smem_tile[a] for a in axis_names if a != tau))


def _plan_key(plan: ProgramPlan, space_axes, axis_names) -> tuple:
    return len(plan.parts), tuple((k.tile_key(space_axes, axis_names), n) for k, n in plan.parts)


# ---------------------------------------------------------------- native tables


def native_table(candidates: Sequence[UKernel], instance: WorkloadInstance):
    """(NativeCands, kernels) for a candidate sequence: reuses the compile
    stage's table when ``candidates`` is its FinalSet for this instance."""
    native = getattr(candidates, "native", None)
    if native is not None and getattr(candidates, "instance", None) == instance:
        return native, candidates
    kernels = list(candidates)
    spec = instance.spec
    space, axes = tuple(spec.space_axes), tuple(spec.space_axes) + tuple(spec.reduce_axes)
    n = len(kernels)
    reg = np.array([[k.reg_tile[a] for a in space] for k in kernels], dtype=np.int64).reshape(n, len(space))
    smem = np.array([[k.smem_tile[a] for a in axes] for k in kernels], dtype=np.int64).reshape(n, len(axes))
    nan = float("nan")
    pad = np.array([nan if k.padding_threshold is None else k.padding_threshold for k in kernels], dtype=np.float64)
    occ = np.array([nan if k.usage_eff is None else k.usage_eff for k in kernels], dtype=np.float64)
    cmr = np.array([nan if k.compute_eff is None else k.compute_eff for k in kernels], dtype=np.float64)
    P, D = C.POINTER(C.c_int64), C.POINTER(C.c_double)
    h = C.c_void_p()
    _lib.check(_native.lib().ftb_cands_from_arrays(
        C.byref(_native.inst_struct(instance)), n, reg.ctypes.data_as(P), smem.ctypes.data_as(P),
        pad.ctypes.data_as(D), occ.ctypes.data_as(D), cmr.ctypes.data_as(D), C.byref(h)))
    return _native.NativeCands(h, len(space), len(axes)), kernels


class PlanPool(list):
    """build_programs' result: a plain list of ProgramPlan that also keeps the
    native candidate table, so rank_programs can stream it in C++."""

    native = None
    tau = None
    kernels = None
    instance = None


def plan_pool_size(candidates: Sequence[UKernel], instance: WorkloadInstance) -> int:
    """Number of plans build_programs would return, without building them."""
    if not len(candidates):
        raise EmptyResultError("candidate set is empty", constraint="candidate set",
                               hint="relax the compile-stage filters")
    native, _ = native_table(candidates, instance)
    tau = select_main_axis(instance)
    n = C.c_int64()
    _lib.check(_native.lib().ftb_pool_count(native.h, instance.spec.space_axes.index(tau), C.byref(n)))
    return n.value


def plans_from_rows(rows: np.ndarray, kernels, instance, tau, scores=None) -> list[ProgramPlan]:
    out = []
    for i, r in enumerate(rows):
        parts = ((kernels[int(r[1])], int(r[2])),) if r[0] == 1 else \
            ((kernels[int(r[1])], int(r[2])), (kernels[int(r[3])], int(r[4])))
        out.append(ProgramPlan(parts=parts, shape=instance, tau=tau,
                               sia=None if scores is None else float(scores[i])))
    return out


def build_programs(candidates: Sequence[UKernel], instance: WorkloadInstance) -> list[ProgramPlan]:
    """Every single-tile covering plus every compatible two-tile combination,
    deduplicated, in canonical plan-key order (combine.py:133-194)."""
    if not len(candidates):
        raise EmptyResultError("candidate set is empty", constraint="candidate set",
                               hint="relax the compile-stage filters")
    native, kernels = native_table(candidates, instance)
    tau = select_main_axis(instance)
    ti = instance.spec.space_axes.index(tau)
    L = _native.lib()
    n = C.c_int64()
    _lib.check(L.ftb_pool_count(native.h, ti, C.byref(n)))
    if n.value == 0:
        raise EmptyResultError(
            f"no uKernel combination covers axis '{tau}' (extent {instance.extent(tau)})",
            constraint="main-axis coverage", hint="relax the compile-stage filters to admit more tile sizes")
    rows = np.zeros((n.value, 5), dtype=np.int64)
    got = C.c_int64()
    _lib.check(L.ftb_pool_export(native.h, ti, n.value, rows.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(got)))
    pool = PlanPool(plans_from_rows(rows, kernels, instance, tau))
    extent = instance.extent(tau)
    for plan in pool:
        if plan.tau_coverage != extent:
            raise InternalError(f"plan covers {plan.tau_coverage} on axis '{tau}', expected {extent}")
    pool.native, pool.tau, pool.kernels, pool.instance = native, tau, kernels, instance
    pool._frozen_len = len(pool)
    return pool
