"""uKernels and hardware-aligned candidate enumeration (drop-in for
mktune.ukernel, ukernel.py:1-437).

``enumerate_ukernels`` runs in the C++ planner (libftb.so) and returns the
same canonical, columnar ``CandidateSet``: lexicographic by (register-tile
vector, shared-memory-tile vector), cap truncation in that order. On a
descriptor carrying the tcgen05 extension the set is additionally restricted
to tcgen05-legal tiles (the B200 mode; see hardware.py).
"""

from __future__ import annotations

import ctypes as C
import logging
import math
from dataclasses import dataclass
from typing import Iterator, Mapping, Sequence

import numpy as np

from .. import _lib
from . import _native
from .errors import CapacityError, InputError, MissingMetricsError
from .hardware import HardwareDescriptor
from .workload import WorkloadInstance, ceil_div

logger = logging.getLogger(__name__)

DEFAULT_CANDIDATE_CAP = 1 << 21


@dataclass
class UKernel:
    """A tile configuration (register tiles inside shared-memory tiles) plus
    the three per-instance metrics the compile stage caches on it."""

    reg_tile: dict
    smem_tile: dict
    padding_threshold: float | None = None
    usage_eff: float | None = None
    compute_eff: float | None = None

    def tile_key(self, space_axes: Sequence[str], axis_names: Sequence[str]) -> tuple:
        return (tuple(self.reg_tile[a] for a in space_axes), tuple(self.smem_tile[a] for a in axis_names))


def divisors(n: int) -> list[int]:
    if n < 1:
        raise InputError(f"divisors() needs a positive integer, got {n}")
    small = [d for d in range(1, math.isqrt(n) + 1) if n % d == 0]
    return small + [n // d for d in reversed(small) if d * d != n]


def _is_prime(n: int) -> bool:
    return n >= 2 and all(n % d for d in range(2, math.isqrt(n) + 1))


def default_major_axis(spec) -> str:
    """The output's innermost (row-major contiguous) axis."""
    return spec.output_access.axes[-1]


def reg_tile_candidates(axis_extent: int, align_elems: int = 8) -> list[int]:
    if axis_extent < 1:
        raise InputError(f"axis extent must be >= 1, got {axis_extent}")
    vals = set(divisors(axis_extent))
    if axis_extent > align_elems and _is_prime(axis_extent):
        vals |= set(divisors(axis_extent - 1)) | set(divisors(axis_extent + 1))
    return sorted(vals)


def space_tile_options(extent: int, reg: int, align_elems: int, is_major: bool) -> list[int]:
    step = math.lcm(reg, align_elems) if is_major else reg
    return [step * m for m in range(1, ceil_div(extent, step) + 1)]


def reduce_tile_options(extent: int, align_elems: int) -> list[int]:
    if extent < align_elems:
        return [align_elems]
    return list(range(align_elems, extent // align_elems * align_elems + 1, align_elems))


def staged_footprint_bytes(spec, smem_tile: Mapping) -> int:
    total = 0
    for acc in spec.input_accesses:
        total += math.prod(smem_tile[a] for a in acc.axes)
    return total * spec.elem_bytes


def check_ukernel(k: UKernel, instance: WorkloadInstance, hw: HardwareDescriptor, major_axis: str | None = None) -> None:
    spec = instance.spec
    major = major_axis or default_major_axis(spec)
    for s in spec.space_axes:
        if k.smem_tile[s] % k.reg_tile[s]:
            raise InputError(
                f"register tile {k.reg_tile[s]} does not divide shared-memory tile {k.smem_tile[s]} on axis '{s}'",
                field=s,
            )
    if k.smem_tile[major] % hw.align_elems:
        raise InputError(
            f"major-axis tile {k.smem_tile[major]} is not a multiple of align_elems={hw.align_elems}", field=major
        )
    fp = staged_footprint_bytes(spec, k.smem_tile)
    if fp > hw.smem_per_core_bytes:
        raise InputError(
            f"staged footprint {fp} B exceeds shared memory capacity {hw.smem_per_core_bytes} B",
            field="smem_per_core_bytes",
        )


def smem_tile_candidates(reg_tile: Mapping, instance: WorkloadInstance, hw: HardwareDescriptor,
                         major_axis: str | None = None) -> list[dict]:
    """Shared-memory tiles valid for one register tile, canonical order (scalar API)."""
    spec = instance.spec
    major = major_axis or default_major_axis(spec)
    axes = list(spec.space_axes) + list(spec.reduce_axes)
    opts = [space_tile_options(instance.extent(a), reg_tile[a], hw.align_elems, a == major) for a in spec.space_axes]
    opts += [reduce_tile_options(instance.extent(a), hw.align_elems) for a in spec.reduce_axes]
    lows = [o[0] for o in opts]
    out: list[dict] = []
    cur = list(lows)

    def rec(d: int) -> None:
        if d == len(axes):
            out.append(dict(zip(axes, cur)))
            return
        for v in opts[d]:
            probe = cur[:d] + [v] + lows[d + 1:]
            if staged_footprint_bytes(spec, dict(zip(axes, probe))) > hw.smem_per_core_bytes:
                break  # footprint is monotone: every larger value overflows too
            cur[d] = v
            rec(d + 1)
        cur[d] = lows[d]

    rec(0)
    return out


class CandidateSet:
    """Columnar candidates for one instance (rows of ``reg`` / ``smem``);
    metric columns are attached by the metrics and filter stages."""

    def __init__(self, instance, hw, major_axis, reg, smem, truncated=False, columns=None):
        self.instance = instance
        self.hw = hw
        self.major_axis = major_axis
        self.reg = reg
        self.smem = smem
        self.truncated = truncated
        self.columns = {} if columns is None else columns

    @property
    def space_axes(self) -> tuple[str, ...]:
        return self.instance.spec.space_axes

    @property
    def axis_names(self) -> tuple[str, ...]:
        return tuple(self.instance.spec.space_axes) + tuple(self.instance.spec.reduce_axes)

    def __len__(self) -> int:
        return self.reg.shape[0]

    def __getitem__(self, i: int) -> UKernel:
        k = UKernel(
            reg_tile={a: int(v) for a, v in zip(self.space_axes, self.reg[i])},
            smem_tile={a: int(v) for a, v in zip(self.axis_names, self.smem[i])},
        )
        cols = self.columns
        if "pad_num" in cols:
            k.padding_threshold = float(cols["pad_num"][i] / cols["pad_den"][i])
            k.usage_eff = float(cols["blocks"][i] / cols["occ_den"][i])
        if "cmr" in cols:
            k.compute_eff = float(cols["cmr"][i])
        return k

    def __iter__(self) -> Iterator[UKernel]:
        return (self[i] for i in range(len(self)))

    def column(self, name: str) -> np.ndarray:
        try:
            return self.columns[name]
        except KeyError:
            raise MissingMetricsError(f"metric column '{name}' has not been computed") from None

    def subset(self, index) -> "CandidateSet":
        return CandidateSet(
            self.instance, self.hw, self.major_axis, self.reg[index], self.smem[index],
            truncated=self.truncated, columns={k: v[index] for k, v in self.columns.items()},
        )

    def tile_keys(self) -> list[tuple]:
        return [(tuple(map(int, r)), tuple(map(int, s))) for r, s in zip(self.reg, self.smem)]

    @classmethod
    def from_ukernels(cls, instance, hw, kernels: Sequence[UKernel], major_axis: str | None = None) -> "CandidateSet":
        spec = instance.spec
        axes = tuple(spec.space_axes) + tuple(spec.reduce_axes)
        reg = np.array([[k.reg_tile[a] for a in spec.space_axes] for k in kernels], dtype=np.int64)
        smem = np.array([[k.smem_tile[a] for a in axes] for k in kernels], dtype=np.int64)
        return cls(instance, hw, major_axis or default_major_axis(spec),
                   reg.reshape(len(kernels), len(spec.space_axes)), smem.reshape(len(kernels), len(axes)))


def enumerate_ukernels(instance: WorkloadInstance, hw: HardwareDescriptor, cap: int | None = DEFAULT_CANDIDATE_CAP,
                       major_axis: str | None = None) -> CandidateSet:
    """Hardware-aligned candidates for one bound shape (C++ planner)."""
    spec = instance.spec
    major = major_axis or default_major_axis(spec)
    if major not in spec.space_axes:
        raise InputError(f"major axis '{major}' is not a space axis", field="major_axis")
    L = _native.lib()
    h = C.c_void_p()
    tr = C.c_int32()
    _lib.check(L.ftb_enumerate(C.byref(_native.hw_struct(hw)), C.byref(_native.inst_struct(instance, major)),
                               -1 if cap is None else int(cap), C.byref(h), C.byref(tr)))
    nc = _native.NativeCands(h, len(spec.space_axes), len(spec.space_axes) + len(spec.reduce_axes))
    try:
        reg, smem, _, _ = nc.arrays(metrics=False)
    finally:
        nc.close()
    if tr.value:
        logger.warning("candidate enumeration for %s hit the cap of %d; truncated in canonical order",
                       instance.binding_key() or spec.name, cap)
    return CandidateSet(instance, hw, major, reg, smem, truncated=bool(tr.value))


__all__ = [
    "DEFAULT_CANDIDATE_CAP", "UKernel", "divisors", "default_major_axis", "reg_tile_candidates",
    "space_tile_options", "reduce_tile_options", "staged_footprint_bytes", "check_ukernel",
    "smem_tile_candidates", "CandidateSet", "enumerate_ukernels", "CapacityError",
]
