"""ctypes binding of libftb.so (include/ftb.h).

The shared library is built in-tree by ``paper_2407_21418_b200/csrc/Makefile``
(``__graft_entry__.build()``). There is no fallback: if the library is missing
every entry point raises, so no Python/CPU path can silently stand in for the
CUDA executor or the C++ planner.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libftb.so"
# FTB_LIB: load another build of the library, e.g. the trace build
# (make -C paper_2407_21418_b200/csrc trace -> libftb_trace.so) for the
# phase-trace scripts under scripts/.
if os.environ.get("FTB_LIB"):
    LIB_PATH = Path(os.environ["FTB_LIB"]).resolve()

MAX_AXES = 8

FTB_OK = 0
FTB_EMPTY_RESULT = 1
FTB_INPUT_ERROR = 2
FTB_INTERNAL_ERROR = 3
FTB_CAPACITY_ERROR = 4
FTB_MISSING_METRICS = 5
FTB_CUDA_ERROR = 6

OP_DENSE, OP_BMM = 0, 1
B_KN, B_NK = 0, 1
DT_BF16, DT_F32 = 0, 1
ACT_NONE, ACT_GELU = 0, 1


class Program(C.Structure):
    _fields_ = [
        ("n_space", C.c_int32),
        ("n_reduce", C.c_int32),
        ("tau", C.c_int32),
        ("n_parts", C.c_int32),
        ("reg", (C.c_int64 * MAX_AXES) * 2),
        ("smem", (C.c_int64 * MAX_AXES) * 2),
        ("count", C.c_int64 * 2),
        ("sia", C.c_double),
    ]


class GemmDesc(C.Structure):
    _fields_ = [
        ("op", C.c_int32),
        ("batch", C.c_int32),
        ("M", C.c_int64),
        ("N", C.c_int64),
        ("K", C.c_int64),
        ("A", C.c_void_p),
        ("lda", C.c_int64),
        ("a_batch_stride", C.c_int64),
        ("B", C.c_void_p),
        ("ldb", C.c_int64),
        ("b_batch_stride", C.c_int64),
        ("C", C.c_void_p),
        ("ldc", C.c_int64),
        ("c_batch_stride", C.c_int64),
        ("b_layout", C.c_int32),
        ("in_dtype", C.c_int32),
        ("out_dtype", C.c_int32),
        ("orientation", C.c_int32),
        ("bias", C.c_void_p),
        ("bias_dtype", C.c_int32),
        ("activation", C.c_int32),
    ]


class ExecInfo(C.Structure):
    _fields_ = [
        ("n_work", C.c_int64),
        ("n_ctas", C.c_int64),
        ("n_problems", C.c_int64),
        ("mma_flops", C.c_int64),
        ("true_flops", C.c_int64),
        ("covered_out", C.c_int64),
        ("true_out", C.c_int64),
        ("kernel", C.c_int32),
    ]


_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib() -> C.CDLL:
    """Load libftb.so once; raise loudly when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise LibraryMissing(
            f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_2407_21418_b200/csrc)"
        )
    L = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "ftb_last_error": (C.c_size_t, [C.c_char_p, C.c_size_t]),
        "ftb_last_error_field": (C.c_size_t, [C.c_char_p, C.c_size_t]),
        "ftb_exec_create": (i32, [C.POINTER(GemmDesc), C.POINTER(Program), i32, C.POINTER(vp)]),
        "ftb_exec_launch": (i32, [vp, vp]),
        "ftb_exec_get_info": (i32, [vp, C.POINTER(ExecInfo)]),
        "ftb_exec_export_table": (i32, [vp, C.POINTER(i32), i64, C.POINTER(i64)]),
        "ftb_exec_destroy": (None, [vp]),
        "ftb_lower": (
            i32,
            [C.POINTER(GemmDesc), C.POINTER(Program), i32, C.POINTER(i32), i64, C.POINTER(i64),
             C.POINTER(ExecInfo)],
        ),
        "ftb_device_sm_count": (i32, []),
        "ftb_exec_set_trace": (i32, [vp, i32]),
        "ftb_exec_read_trace": (i32, [vp, C.POINTER(C.c_uint64), i64, C.POINTER(i64)]),
        "ftb_exec_get_config": (i32, [vp, C.POINTER(i32)]),
        "ftb_test_occupy_sms": (i32, [i32, vp, i64, vp]),
    }
    optional = {"ftb_test_occupy_sms"}  # test hook: absent from older builds used in A/B runs
    for name, (res, args) in sig.items():
        if name in optional and not hasattr(L, name):
            continue
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def declared_symbols() -> list[str]:
    """Every function name declared in include/ftb.h (for the export test)."""
    import re

    hdr = (_HERE.parent / "include" / "ftb.h").read_text()
    body = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(ftb_[a-z0-9_]+)\s*\(", body)))


def last_error() -> tuple[str, str]:
    L = lib()
    buf = C.create_string_buffer(4096)
    L.ftb_last_error(buf, 4096)
    fbuf = C.create_string_buffer(256)
    L.ftb_last_error_field(fbuf, 256)
    return buf.value.decode(errors="replace"), fbuf.value.decode(errors="replace")


def check(status: int) -> None:
    """Raise the mktune exception class that matches a status code (errors.py:10-47)."""
    if status == FTB_OK:
        return
    from .mktune import errors as E

    msg, field = last_error()
    raise E.TunerError.from_status(status, msg, field)


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0", "false", "False")
