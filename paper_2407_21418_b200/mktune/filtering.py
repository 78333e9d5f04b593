"""Compile-stage filtering (drop-in for mktune.filtering, filtering.py:1-405).

``compile_shape`` and ``compile_stage`` run the whole per-shape pipeline
(enumerate -> annotate -> cross-pick -> set-bound -> multi-axis filter ->
relaxation ladder) in the C++ planner and return the reference's
``ShapeResult`` / ``CompileResult``. The candidate and bundle lists are lazy
sequences: UKernel / MetricBundle objects are built on first access, which
removes the reference's per-survivor Python loop (filtering.py:320-331)
from the critical path. The individual passes (``cross_pick``,
``set_bound``, ``multi_axis_filter``, ``retention_steps``) are also provided
over ``CandidateSet`` in numpy for callers that compose them by hand.
"""

from __future__ import annotations

import ctypes as C
import logging
from collections.abc import Sequence as SequenceABC
from dataclasses import dataclass, replace
from fractions import Fraction
from typing import Sequence

import numpy as np

from .. import _lib
from . import _native
from .errors import InputError
from .metrics import (
    DEFAULT_PSI,
    DEFAULT_REST_REGS,
    MetricBundle,
    annotate_geometry,
    annotate_intensity,
    annotate_registers,
)
from .ukernel import DEFAULT_CANDIDATE_CAP, CandidateSet, UKernel
from .workload import OperatorSpec, WorkloadInstance, ceil_div

logger = logging.getLogger(__name__)

_MAX_DEN = 10_000
DEFAULT_FINAL_CEILING = 256
_MAX_WIDENING = 2_000


def _as_fraction(value, name: str) -> Fraction:
    if isinstance(value, Fraction):
        f = value
    else:
        try:
            f = Fraction(str(value))
        except (ValueError, ZeroDivisionError) as exc:
            raise InputError(f"sweep parameter '{name}' is not a number: {value!r}", field=name) from exc
    if not 0 <= f <= 1:
        raise InputError(f"sweep parameter '{name}' must lie in [0, 1], got {f}", field=name)
    if f.denominator > _MAX_DEN:
        raise InputError(
            f"sweep parameter '{name}' needs denominator <= {_MAX_DEN} (use decimals with at most 4 places), got {f}",
            field=name,
        )
    return f


_SWEEP_FIELDS = ("eps_min", "eps_max", "lam_min", "lam_max", "eps_step", "lam_step")


@dataclass(frozen=True)
class SweepParams:
    """Padding/occupancy cross-sweep bounds and strides, exact rationals."""

    eps_min: Fraction = Fraction(1, 2)
    eps_max: Fraction = Fraction(19, 20)
    lam_min: Fraction = Fraction(9, 10)
    lam_max: Fraction = Fraction(19, 20)
    eps_step: Fraction = Fraction(1, 100)
    lam_step: Fraction = Fraction(1, 1000)

    def __post_init__(self):
        for n in _SWEEP_FIELDS:
            object.__setattr__(self, n, _as_fraction(getattr(self, n), n))
        if not self.eps_min < self.eps_max:
            raise InputError("sweep requires eps_min < eps_max", field="eps_min")
        if not self.lam_min < self.lam_max:
            raise InputError("sweep requires lam_min < lam_max", field="lam_min")
        if self.eps_step <= 0 or self.lam_step <= 0:
            raise InputError("sweep strides must be positive", field="eps_step")

    @property
    def num_steps(self) -> int:
        return 1 + min(int((self.eps_max - self.eps_min) / self.eps_step),
                       int((self.lam_max - self.lam_min) / self.lam_step))

    def point(self, step: int) -> tuple[Fraction, Fraction]:
        return self.eps_min + (step - 1) * self.eps_step, self.lam_max - (step - 1) * self.lam_step

    def widened(self, strides: int) -> "SweepParams":
        return replace(self, eps_min=max(Fraction(0), self.eps_min - strides * self.eps_step),
                       lam_min=max(Fraction(0), self.lam_min - strides * self.lam_step))

    def to_doc(self) -> dict:
        return {n: str(getattr(self, n)) for n in _SWEEP_FIELDS}

    @classmethod
    def from_doc(cls, doc: dict) -> "SweepParams":
        return cls(**{k: Fraction(v) for k, v in doc.items()})


def retention_steps(cs: CandidateSet, sweep: SweepParams) -> np.ndarray:
    """First 1-based sweep step at which each candidate clears both
    thresholds, 0 if never (closed form; exact int64 cross-multiplication)."""
    annotate_geometry(cs)
    c = cs.columns
    en, ed = sweep.eps_min.numerator, sweep.eps_min.denominator
    sn, sd = sweep.eps_step.numerator, sweep.eps_step.denominator
    ln, ld = sweep.lam_max.numerator, sweep.lam_max.denominator
    tn, td = sweep.lam_step.numerator, sweep.lam_step.denominator
    pad_last = 1 + ((c["pad_num"] * ed - en * c["pad_den"]) * sd) // (c["pad_den"] * ed * sn)
    occ_first = np.maximum(1 + ceil_div((ln * c["occ_den"] - c["blocks"] * ld) * td, c["occ_den"] * ld * tn), 1)
    hit = occ_first <= np.minimum(pad_last, sweep.num_steps)
    return np.where(hit, occ_first, 0).astype(np.int64)


def cross_pick(candidates: CandidateSet, instance: WorkloadInstance, hw, sweep: SweepParams | None = None) -> CandidateSet:
    sweep = sweep or SweepParams()
    annotate_geometry(candidates)
    if "footprint" not in candidates.columns:
        col = {a: j for j, a in enumerate(candidates.axis_names)}
        fp = np.zeros(len(candidates), dtype=np.int64)
        for acc in instance.spec.input_accesses:
            term = np.ones(len(candidates), dtype=np.int64)
            for a in acc.axes:
                term = term * candidates.smem[:, col[a]]
            fp += term
        candidates.columns["footprint"] = fp * instance.spec.elem_bytes
    steps = retention_steps(candidates, sweep)
    keep = (candidates.columns["footprint"] <= hw.smem_per_core_bytes) & (steps > 0)
    out = candidates.subset(np.flatnonzero(keep))
    out.columns["retained_step"] = steps[keep]
    return out


def set_bound(kcross: CandidateSet, instance: WorkloadInstance, hw, rest_regs: int = DEFAULT_REST_REGS) -> CandidateSet:
    annotate_geometry(kcross)
    annotate_registers(kcross, rest_regs)
    bound = np.minimum(ceil_div(kcross.columns["blocks"], hw.num_cores), hw.default_active_blocks)
    keep = kcross.columns["regs_in_block"] * bound <= hw.regs_per_core
    out = kcross.subset(np.flatnonzero(keep))
    out.columns["block_bound"] = bound[keep]
    return out


def multi_axis_filter(kfilter: CandidateSet, instance: WorkloadInstance, hw, psi: float = DEFAULT_PSI) -> CandidateSet:
    annotate_intensity(kfilter)
    return kfilter.subset(np.flatnonzero(kfilter.columns["saturated"] & (kfilter.columns["cmr"] >= psi)))


def _saturation_only(kfilter: CandidateSet) -> CandidateSet:
    annotate_intensity(kfilter)
    return kfilter.subset(np.flatnonzero(kfilter.columns["saturated"]))


@dataclass
class FilterParams:
    sweep: SweepParams
    psi: float = DEFAULT_PSI
    rest_regs: int = DEFAULT_REST_REGS
    candidate_cap: int | None = DEFAULT_CANDIDATE_CAP
    final_ceiling: int | None = DEFAULT_FINAL_CEILING  # declared, never applied (as in the reference)
    major_axis: str | None = None

    @classmethod
    def default(cls) -> "FilterParams":
        return cls(sweep=SweepParams())


@dataclass
class ShapeResult:
    binding: dict
    candidates: Sequence
    bundles: Sequence
    retained_steps: list
    counts: dict
    relaxation: str
    truncated: bool
    sweep_used: SweepParams


class FinalSet(SequenceABC):
    """The final candidates of one shape as a lazy sequence of UKernel
    (metrics cached on each, as filtering.py:326-329 does). Keeps the native
    table so build_programs / rank can stay in C++."""

    def __init__(self, instance, native, reg, smem, icol, fcol):
        self.instance = instance
        self.native = native  # _native.NativeCands (owning)
        self.reg, self.smem, self.icol, self.fcol = reg, smem, icol, fcol
        spec = instance.spec
        self._space = tuple(spec.space_axes)
        self._axes = self._space + tuple(spec.reduce_axes)
        self._cache: dict[int, UKernel] = {}

    def __len__(self):
        return self.reg.shape[0]

    def _make(self, i: int) -> UKernel:
        k = self._cache.get(i)
        if k is None:
            ic = self.icol[i]
            k = UKernel(
                reg_tile={a: int(v) for a, v in zip(self._space, self.reg[i])},
                smem_tile={a: int(v) for a, v in zip(self._axes, self.smem[i])},
                padding_threshold=float(Fraction(int(ic[0]), int(ic[1]))),
                usage_eff=float(Fraction(int(ic[2]), int(ic[3]))),
                compute_eff=float(self.fcol[i, 0]),
            )
            self._cache[i] = k
        return k

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._make(j) for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return self._make(i)

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self):
        return f"FinalSet({len(self)} uKernels)"


class BundleList(SequenceABC):
    def __init__(self, final: FinalSet):
        self.f = final

    def __len__(self):
        return len(self.f)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        ic, fc = self.f.icol[i], self.f.fcol[i]
        return MetricBundle(
            pad=Fraction(int(ic[0]), int(ic[1])), occ=Fraction(int(ic[2]), int(ic[3])),
            regs_in_block=int(ic[4]), saturated=bool(ic[5]), cmr=float(fc[0]),
            mem_latency_s=float(fc[1]), blocks_needed=int(ic[2]),
        )

    def __eq__(self, other):
        return list(self) == list(other)


def _sweep_from(report) -> SweepParams:
    f = [_native.frac_from(report.sweep_used[i]) for i in range(6)]
    return SweepParams(*f)


def compile_shape(instance: WorkloadInstance, hw, params: FilterParams | None = None) -> ShapeResult:
    """Per-shape pipeline with the relaxation ladder, in the C++ planner."""
    params = params or FilterParams.default()
    L = _native.lib()
    h = C.c_void_p()
    rep = _native.Report()
    _lib.check(L.ftb_compile_shape(
        C.byref(_native.hw_struct(hw)), C.byref(_native.inst_struct(instance, params.major_axis)),
        C.byref(_native.params_struct(params)), C.byref(h), C.byref(rep),
    ))
    spec = instance.spec
    nc = _native.NativeCands(h, len(spec.space_axes), len(spec.space_axes) + len(spec.reduce_axes))
    reg, smem, icol, fcol = nc.arrays(metrics=True)
    if rep.truncated:
        logger.warning("candidate enumeration for %s hit the cap of %s; truncated in canonical order",
                       instance.binding_key() or spec.name, params.candidate_cap)
    final = FinalSet(instance, nc, reg, smem, icol, fcol)
    res = ShapeResult(
        binding=dict(instance.bindings),
        candidates=final,
        bundles=BundleList(final),
        retained_steps=[int(v) for v in icol[:, 6]],
        counts={"align": rep.n_align, "cross": rep.n_cross, "filter": rep.n_filter, "final": rep.n_final},
        relaxation=_native.relaxation_name(rep.relaxation, rep.widen),
        truncated=bool(rep.truncated),
        sweep_used=_sweep_from(rep),
    )
    res.tuning_seconds = rep.seconds  # provenance (not in the reference)
    return res


@dataclass
class CompileResult:
    spec: OperatorSpec
    hw: object
    params: FilterParams
    sections: list


def default_bindings(spec: OperatorSpec) -> list[dict]:
    from itertools import product

    dyn = spec.dynamic_axes
    spans = [range(spec.axis(a).range[0], spec.axis(a).range[1] + 1) for a in dyn]
    return [dict(zip(dyn, combo)) for combo in product(*spans)]


def compile_stage(spec: OperatorSpec, hw, params: FilterParams | None = None,
                  bindings: Sequence[dict] | None = None, workers: int = 1) -> CompileResult:
    """compile_shape over every binding, results in binding order. Shapes run
    on a host thread pool (the C++ planner releases the GIL), so the output
    is identical at any ``workers``."""
    params = params or FilterParams.default()
    if bindings is None:
        bindings = [{}] if not spec.dynamic_axes else default_bindings(spec)
    if not bindings:
        raise InputError("no shape bindings requested", field="bindings")

    def one(b):
        return compile_shape(WorkloadInstance(spec=spec, bindings=dict(b)), hw, params)

    if workers > 1 and len(bindings) > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=workers) as ex:
            sections = list(ex.map(one, bindings))
    else:
        sections = [one(b) for b in bindings]
    return CompileResult(spec=spec, hw=hw, params=params, sections=sections)
