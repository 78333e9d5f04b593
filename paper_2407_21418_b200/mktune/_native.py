"""Marshalling between the facade's value types and the C++ planner
(libftb.so, include/ftb.h). Internal to the facade."""

from __future__ import annotations

import ctypes as C
from fractions import Fraction

import numpy as np

from .. import _lib
from ..execute import program_struct
from .errors import InputError

MAX_AXES = _lib.MAX_AXES
MAX_INPUTS = 4


class Hw(C.Structure):
    _fields_ = [(f, C.c_int64) for f in (
        "num_cores", "regs_per_core", "smem_per_core_bytes", "global_bw_bytes_per_s",
        "shared_bw_bytes_per_s", "peak_flops", "default_active_blocks", "active_blocks_per_core", "align_elems",
    )] + [("legality", C.c_int32), ("reserved", C.c_int32)] + [(f, C.c_int64) for f in (
        "tmem_columns", "mma_m_max", "mma_n_step", "mma_n_max", "tma_swizzle_bytes")]


class Inst(C.Structure):
    _fields_ = [
        ("n_space", C.c_int32), ("n_reduce", C.c_int32), ("major", C.c_int32), ("n_inputs", C.c_int32),
        ("input_naxes", C.c_int32 * MAX_INPUTS),
        ("input_axes", (C.c_int32 * MAX_AXES) * MAX_INPUTS),
        ("elem_bytes", C.c_int32), ("flops_per_point", C.c_int32),
        ("extent", C.c_int64 * MAX_AXES),
        ("dynamic", C.c_int32 * MAX_AXES),
        ("axis_name", (C.c_char * 16) * MAX_AXES),
    ]


class Frac(C.Structure):
    _fields_ = [("num", C.c_int64), ("den", C.c_int64)]


class Params(C.Structure):
    _fields_ = [(n, Frac) for n in ("eps_min", "eps_max", "lam_min", "lam_max", "eps_step", "lam_step")] + [
        ("psi", C.c_double), ("rest_regs", C.c_int64), ("candidate_cap", C.c_int64),
    ]


class Coeffs(C.Structure):
    _fields_ = [("c0", C.c_double), ("c1", C.c_double), ("c2", C.c_double)]


class Report(C.Structure):
    _fields_ = [
        ("n_align", C.c_int64), ("n_cross", C.c_int64), ("n_filter", C.c_int64), ("n_final", C.c_int64),
        ("relaxation", C.c_int32), ("widen", C.c_int32), ("truncated", C.c_int32), ("tau", C.c_int32),
        ("sweep_used", Frac * 6), ("stage", C.c_int32), ("reserved", C.c_int32), ("seconds", C.c_double),
    ]


_SIGS_DONE = False


def lib():
    global _SIGS_DONE
    L = _lib.lib()
    if not _SIGS_DONE:
        vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int64)
        sig = {
            "ftb_enumerate": (i32, [C.POINTER(Hw), C.POINTER(Inst), i64, C.POINTER(vp), C.POINTER(i32)]),
            "ftb_compile_shape": (i32, [C.POINTER(Hw), C.POINTER(Inst), C.POINTER(Params), C.POINTER(vp), C.POINTER(Report)]),
            "ftb_cands_from_arrays": (i32, [C.POINTER(Inst), i64, ip, ip, dp, dp, dp, C.POINTER(vp)]),
            "ftb_cands_size": (i64, [vp]),
            "ftb_cands_export": (i32, [vp, ip, ip, ip, dp]),
            "ftb_cands_destroy": (None, [vp]),
            "ftb_select_main_axis": (i32, [C.POINTER(Inst), C.POINTER(i32)]),
            "ftb_pool_count": (i32, [vp, i32, C.POINTER(i64)]),
            "ftb_pool_export": (i32, [vp, i32, i64, ip, C.POINTER(i64)]),
            "ftb_rank_topk": (i32, [vp, i32, C.POINTER(Coeffs), i32, i32, ip, dp, C.POINTER(i32)]),
            "ftb_plan_batch": (i32, [C.POINTER(Hw), C.POINTER(Inst), i32, C.POINTER(Params), C.POINTER(Coeffs), i32,
                                     C.POINTER(_lib.Program), C.POINTER(Report), C.POINTER(i32)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _SIGS_DONE = True
    return L


def hw_struct(hw) -> Hw:
    h = Hw()
    for f, _ in Hw._fields_[:9]:
        setattr(h, f, int(getattr(hw, f)))
    h.legality = 1 if getattr(hw, "tmem_columns", None) is not None else 0
    if h.legality:  # the tile rules derive from these (planner.cpp tcgen05_legal)
        h.tmem_columns = int(hw.tmem_columns)
        h.mma_m_max = int(max(hw.mma_m_atoms))
        h.mma_n_step = int(hw.mma_n_step)
        h.mma_n_max = int(hw.mma_n_max)
        h.tma_swizzle_bytes = int(hw.tma_swizzle_bytes)
    return h


def axis_order(spec) -> tuple:
    return tuple(spec.space_axes) + tuple(spec.reduce_axes)


def inst_struct(instance, major_axis: str | None = None) -> Inst:
    spec = instance.spec
    axes = axis_order(spec)
    if len(axes) > MAX_AXES:
        raise InputError(f"at most {MAX_AXES} axes are supported by the native planner", field="axes")
    ins = spec.input_accesses
    if len(ins) > MAX_INPUTS:
        raise InputError(f"at most {MAX_INPUTS} input accesses are supported by the native planner", field="accesses")
    major = major_axis or spec.output_access.axes[-1]
    if major not in spec.space_axes:
        raise InputError(f"major axis '{major}' is not a space axis", field="major_axis")
    s = Inst()
    s.n_space = len(spec.space_axes)
    s.n_reduce = len(spec.reduce_axes)
    s.major = spec.space_axes.index(major)
    s.n_inputs = len(ins)
    for q, acc in enumerate(ins):
        s.input_naxes[q] = len(acc.axes)
        for d, ax in enumerate(acc.axes):
            s.input_axes[q][d] = axes.index(ax)
    s.elem_bytes = spec.elem_bytes
    s.flops_per_point = spec.flops_per_point
    for d, ax in enumerate(axes):
        s.extent[d] = instance.extent(ax)
        s.dynamic[d] = 1 if spec.axis(ax).is_dynamic else 0
        nm = ax.encode()
        if len(nm) > 16:
            raise InputError(f"axis name '{ax}' longer than 16 bytes", field="axes")
        s.axis_name[d].value = nm
    return s


def params_struct(params) -> Params:
    p = Params()
    sw = params.sweep
    for n in ("eps_min", "eps_max", "lam_min", "lam_max", "eps_step", "lam_step"):
        f = Fraction(getattr(sw, n))
        setattr(p, n, Frac(f.numerator, f.denominator))
    p.psi = float(params.psi)
    p.rest_regs = int(params.rest_regs)
    p.candidate_cap = -1 if params.candidate_cap is None else int(params.candidate_cap)
    return p


def coeffs_struct(coeffs) -> Coeffs:
    return Coeffs(float(coeffs.c0), float(coeffs.c1), float(coeffs.c2))


class NativeCands:
    """Owning handle of an ftb_cands table."""

    def __init__(self, handle: C.c_void_p, n_space: int, n_axes: int):
        self.h = handle
        self.ns = n_space
        self.na = n_axes

    def __len__(self):
        return int(lib().ftb_cands_size(self.h))

    def arrays(self, metrics: bool = True):
        n = len(self)
        reg = np.zeros((n, self.ns), dtype=np.int64)
        smem = np.zeros((n, self.na), dtype=np.int64)
        icol = np.zeros((n, 7), dtype=np.int64) if metrics else None
        fcol = np.zeros((n, 2), dtype=np.float64) if metrics else None
        P = C.POINTER(C.c_int64)
        _lib.check(lib().ftb_cands_export(
            self.h, reg.ctypes.data_as(P), smem.ctypes.data_as(P),
            icol.ctypes.data_as(P) if metrics else None,
            fcol.ctypes.data_as(C.POINTER(C.c_double)) if metrics else None,
        ))
        return reg, smem, icol, fcol

    def close(self):
        if self.h:
            lib().ftb_cands_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def frac_from(f: Frac) -> Fraction:
    return Fraction(f.num, f.den)


RELAXATION = {0: "none", 1: "drop-intensity", 2: "drop-saturation", 3: "widen-sweep-{}", 4: "drop-sweep"}


def relaxation_name(code: int, widen: int) -> str:
    s = RELAXATION[code]
    return s.format(widen) if code == 3 else s


__all__ = ["program_struct"]
