"""Executor front end: ProgramPlan -> tile-schedule table -> one persistent
sm_100a kernel launch (libftb.so, include/ftb.h).

This is the "execute" half the reference does not have. A plan is
the reference's ProgramPlan (combine.py:30-55): one or two uKernels with
repetition counts along the main axis tau, uniform tiles elsewhere. Both the
facade's plans (``paper_2407_21418_b200.mktune.combine.ProgramPlan``) and the
reference's own objects are accepted — anything with ``parts``, ``tau`` and
``shape``.

Torch provides device memory and the stream; the kernels, lowering and TMA
descriptors live in libftb.so. Nothing here computes on the CPU: if the
library is missing, calls raise.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

from . import _lib
from ._lib import DT_BF16, DT_F32, OP_BMM, OP_DENSE, B_KN, B_NK, GemmDesc, Program


# --------------------------------------------------------------------- programs


def program_struct(
    n_space: int,
    tau: int,
    parts: Sequence[tuple[Sequence[int], Sequence[int], int]],
    sia: float = 0.0,
) -> Program:
    """Build an ftb_program from ``[(reg_tiles, smem_tiles, count), ...]``.

    ``reg_tiles`` has one entry per space axis, ``smem_tiles`` one per axis
    (space then reduce), in operator axis order.
    """
    g = Program()
    g.n_space = n_space
    g.n_reduce = 1
    g.tau = tau
    g.n_parts = len(parts)
    if not 1 <= len(parts) <= 2:
        raise ValueError("a program has one or two parts")
    for p, (reg, smem, count) in enumerate(parts):
        for a, v in enumerate(reg):
            g.reg[p][a] = int(v)
        for a, v in enumerate(smem):
            g.smem[p][a] = int(v)
        g.count[p] = int(count)
    g.sia = float(sia) if sia is not None else 0.0
    return g


def program_from_plan(plan) -> Program:
    """Convert a ProgramPlan (facade or reference object) to ftb_program."""
    spec = plan.shape.spec
    space = list(spec.space_axes)
    axes = space + list(spec.reduce_axes)
    parts = []
    for k, n in plan.parts:
        parts.append(([k.reg_tile[a] for a in space], [k.smem_tile[a] for a in axes], n))
    return program_struct(len(space), space.index(plan.tau), parts, plan.sia or 0.0)


# --------------------------------------------------------------------- problems


def _dt(t) -> int:
    import torch

    if t.dtype == torch.bfloat16:
        return DT_BF16
    if t.dtype == torch.float32:
        return DT_F32
    raise TypeError(f"unsupported dtype {t.dtype}; use bfloat16 (tcgen05) or float32 (FFMA)")


def gemm_desc(A, B, Cout, b_layout: str = "kn", orientation: int = -1, bias=None,
              activation: str | None = None) -> GemmDesc:
    """Describe ``Cout = act(A @ B + bias)`` for 2-D (Dense) or 3-D
    (BatchMatmul) tensors.

    ``b_layout="kn"``: B is [K, N] (or [b, K, N]) as in the reference's access
    B[k, j]; ``"nk"``: B is given as its [N, K] transpose (nn.Linear weight
    layout). Only the last dimension of each tensor must be contiguous.
    ``bias`` ([N], bf16 or fp32) and ``activation`` (None or ``"gelu"``, the
    erf form of ``torch.nn.functional.gelu``) are fused into the epilogue
    (Dense only).
    """
    d = GemmDesc()
    if b_layout not in ("kn", "nk"):
        raise ValueError(f"b_layout must be 'kn' or 'nk', not {b_layout!r}")
    # The TMA descriptors and the work table are built from these extents, not
    # from the allocations: every operand must agree with them, or the kernel
    # would read past B or write past Cout (torch.matmul raises here too).
    if A.dim() == 2:
        d.op, d.batch = OP_DENSE, 1
        M, K = A.shape
        if B.dim() != 2 or Cout.dim() != 2:
            raise ValueError("Dense needs 2-D A, B and C")
        Kb, N = (B.shape[0], B.shape[1]) if b_layout == "kn" else (B.shape[1], B.shape[0])
        if tuple(Cout.shape) != (M, N):
            raise ValueError(f"C has shape {tuple(Cout.shape)}, expected {(M, N)}")
        d.a_batch_stride = d.b_batch_stride = d.c_batch_stride = 0
        rows = lambda t: t.stride(0)  # noqa: E731
    elif A.dim() == 3:
        d.op = OP_BMM
        d.batch, M, K = A.shape
        if B.dim() != 3 or Cout.dim() != 3:
            raise ValueError("BatchMatmul needs 3-D A, B and C")
        Kb, N = (B.shape[1], B.shape[2]) if b_layout == "kn" else (B.shape[2], B.shape[1])
        if B.shape[0] != d.batch:
            raise ValueError(f"B has batch {B.shape[0]}, A has {d.batch}")
        if tuple(Cout.shape) != (d.batch, M, N):
            raise ValueError(f"C has shape {tuple(Cout.shape)}, expected {(d.batch, M, N)}")
        d.a_batch_stride, d.b_batch_stride, d.c_batch_stride = A.stride(0), B.stride(0), Cout.stride(0)
        rows = lambda t: t.stride(1)  # noqa: E731
    else:
        raise ValueError("A must be 2-D (dense) or 3-D (batch matmul)")
    if Kb != K:
        raise ValueError(f"inner dimensions differ: A has K={K}, B has K={Kb} (b_layout={b_layout!r})")
    for name, t in (("A", A), ("B", B), ("C", Cout)):
        if t.stride(-1) != 1:
            raise ValueError(f"{name} must be contiguous in its last dimension")
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (the executor has no CPU path)")
        if t.device != A.device:
            raise ValueError(f"{name} is on {t.device}, A on {A.device}: one problem lives on one device")
    d.M, d.N, d.K = int(M), int(N), int(K)
    d.A, d.B, d.C = A.data_ptr(), B.data_ptr(), Cout.data_ptr()
    d.lda, d.ldb, d.ldc = rows(A), rows(B), rows(Cout)
    d.b_layout = B_KN if b_layout == "kn" else B_NK
    d.in_dtype = _dt(A)
    if _dt(B) != d.in_dtype:
        raise TypeError("A and B must share a dtype")
    d.out_dtype = _dt(Cout)
    d.orientation = orientation
    if bias is not None:
        if bias.dim() != 1 or bias.shape[0] != d.N or not bias.is_cuda or bias.stride(0) != 1:
            raise ValueError("bias must be a contiguous CUDA vector of length N")
        if bias.device != A.device:
            raise ValueError(f"bias is on {bias.device}, A on {A.device}")
        d.bias = bias.data_ptr()
        d.bias_dtype = _dt(bias)
    if activation not in (None, "none", "gelu"):
        raise ValueError(f"unsupported activation {activation!r} (None or 'gelu')")
    d.activation = _lib.ACT_GELU if activation == "gelu" else _lib.ACT_NONE
    d.device_index = A.device.index if A.device.index is not None else _current_device()
    return d


def _current_device() -> int:
    import torch

    return torch.cuda.current_device()


# --------------------------------------------------------------------- executable


@dataclass
class ExecInfo:
    n_work: int
    n_ctas: int
    n_problems: int
    mma_flops: int
    true_flops: int
    covered_out: int
    true_out: int
    kernel: str

    @property
    def padding_ratio(self) -> float:
        """(covered - true) / covered over the output space."""
        return (self.covered_out - self.true_out) / self.covered_out if self.covered_out else 0.0


class Executable:
    """A lowered, device-resident tile-schedule table for a group of problems.

    ``launch()`` runs all of them in ONE persistent kernel launch; it can be
    captured in a CUDA graph. Buffers must stay alive and keep their
    addresses for the lifetime of the Executable (TMA descriptors embed them).
    """

    def __init__(self, descs: Sequence[GemmDesc], programs: Sequence[Program], keepalive=()):
        import torch

        L = _lib.lib()
        n = len(descs)
        if n != len(programs) or n == 0:
            raise ValueError("need one program per problem")
        devs = {getattr(d, "device_index", None) for d in descs} - {None}
        if len(devs) > 1:
            raise ValueError(f"one table runs on one device; problems span devices {sorted(devs)}")
        # the table, its TMA descriptors and the launch belong to the tensors'
        # device, whatever the caller's current device is
        self.device = torch.device("cuda", devs.pop() if devs else torch.cuda.current_device())
        self._descs = (GemmDesc * n)(*descs)
        self._progs = (Program * n)(*programs)
        self._keep = list(keepalive)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.ftb_exec_create(self._descs, self._progs, n, C.byref(h)))
        self._h = h
        info = _lib.ExecInfo()
        _lib.check(L.ftb_exec_get_info(self._h, C.byref(info)))
        self.info = ExecInfo(
            info.n_work, info.n_ctas, info.n_problems, info.mma_flops, info.true_flops,
            info.covered_out, info.true_out, "tcgen05" if info.kernel == 0 else "ffma",
        )

    def launch(self, stream=None) -> None:
        import torch

        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if s.device != self.device:
            raise ValueError(f"stream is on {s.device}, the table on {self.device}")
        fn = _lib.lib().ftb_exec_launch
        if torch.cuda.current_device() == self.device.index:  # the common case: no device switch needed
            st = fn(self._h, C.c_void_p(s.cuda_stream))
        else:
            with torch.cuda.device(self.device):
                st = fn(self._h, C.c_void_p(s.cuda_stream))
        if st:
            _lib.check(st)

    def config(self) -> dict:
        """Pipeline shape chosen for this table (tcgen05 kernel)."""
        out = (C.c_int32 * 12)()
        _lib.check(_lib.lib().ftb_exec_get_config(self._h, out))
        one = {"stages": out[0], "col_stage_bytes": out[1], "n_acc": out[2], "acc_cols": out[3]}
        pair = {"stages": out[4], "col_stage_bytes": out[5], "n_acc": out[6], "acc_cols": out[7]}
        return {"single": one, "pair": pair, "n_singles": out[8], "n_pairs": out[9],
                "cluster_split": out[10], "workspace_split": bool(out[11])}

    def set_trace(self, enable: bool = True) -> None:
        _lib.check(_lib.lib().ftb_exec_set_trace(self._h, 1 if enable else 0))

    def read_trace(self):
        """(items [n_ctas, 16, 6], kblocks [n_ctas, 64, 2]) of %globaltimer ns
        (0 = not reached); see include/ftb.h ftb_exec_set_trace. Also sets
        ``self.trace_span`` = [n_ctas, 2] (CTA start, end stamps)."""
        import numpy as np

        L = _lib.lib()
        n = C.c_int64()
        _lib.check(L.ftb_exec_read_trace(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint64)
        _lib.check(L.ftb_exec_read_trace(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)), n.value, C.byref(n)))
        per = 16 * 6 + 2 * 64 + 2
        out = out.reshape(-1, per)
        self.trace_span = out[:, -2:]  # per CTA: start, end stamps
        return out[:, : 16 * 6].reshape(-1, 16, 6), out[:, 16 * 6: 16 * 6 + 128].reshape(-1, 64, 2)

    def table(self):
        """The lowered work items as an int32 numpy array [n_work, 8]."""
        import numpy as np

        L = _lib.lib()
        n = C.c_int64()
        _lib.check(L.ftb_exec_export_table(self._h, None, 0, C.byref(n)))
        out = np.zeros((n.value, 8), dtype=np.int32)
        _lib.check(
            L.ftb_exec_export_table(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)), n.value, C.byref(n))
        )
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().ftb_exec_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - destructor timing is GC-dependent
        try:
            self.close()
        except Exception:
            pass


def lower_table(descs: Sequence[GemmDesc], programs: Sequence[Program]):
    """Host-only lowering (no GPU needed): returns (table int32 [n,8], info)."""
    import numpy as np

    L = _lib.lib()
    n = len(descs)
    D = (GemmDesc * n)(*descs)
    P = (Program * n)(*programs)
    cnt = C.c_int64()
    info = _lib.ExecInfo()
    _lib.check(L.ftb_lower(D, P, n, None, 0, C.byref(cnt), C.byref(info)))
    out = np.zeros((cnt.value, 8), dtype=np.int32)
    _lib.check(L.ftb_lower(D, P, n, out.ctypes.data_as(C.POINTER(C.c_int32)), cnt.value, C.byref(cnt),
                           C.byref(info)))
    return out, info


def run_plan(plan, A, B, Cout=None, b_layout: str = "kn", orientation: int = -1, stream=None):
    """Execute one ProgramPlan on device tensors; returns C."""
    import torch

    if Cout is None:
        if A.dim() == 2:
            N = B.shape[1] if b_layout == "kn" else B.shape[0]
            shape = (A.shape[0], N)
        else:
            N = B.shape[2] if b_layout == "kn" else B.shape[1]
            shape = (A.shape[0], A.shape[1], N)
        out_dtype = torch.float32 if A.dtype == torch.float32 else torch.bfloat16
        Cout = torch.empty(shape, dtype=out_dtype, device=A.device)
    ex = Executable([gemm_desc(A, B, Cout, b_layout, orientation)], [program_from_plan(plan)], (A, B, Cout))
    ex.launch(stream)
    return Cout
