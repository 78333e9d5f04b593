"""PyTorch custom ops over the uKernel executor ("PyTorch
wrapper: torch.library ops dense(A,B) -> C, bmm(A,B) -> C, execute_table(...),
fake/meta kernels for shape inference").

    import paper_2407_21418_b200.torch_ops  # registers torch.ops.ftb.*
    C = torch.ops.ftb.dense(A, W, "nk", bias, "gelu")      # act(A @ W^T + bias)
    S = torch.ops.ftb.bmm(Q, K, "nk", "ij")                 # attention scores
    outs = torch.ops.ftb.execute_table([A0, A1], [B0, B1], "nk,kn")        # one launch

Every op plans with the runtime Planner (SIA Top-1, B200 legality, cached
per shape) and runs on the sm_100a executor; there is no CPU path — a
non-CUDA input raises. Operands whose row strides are not TMA-legal (a
multiple of 8 elements, 16-byte aligned base) are first copied into padded
buffers. The fake kernels give output shapes and dtypes for meta / fake
tensors (torch.compile tracing, shape propagation).
"""

from __future__ import annotations

import threading
from typing import List, Optional

import torch

from .execute import Executable, gemm_desc
from .runtime import Planner, bmm_instance, dense_instance

_planner_lock = threading.Lock()
_planner: Planner | None = None


def planner() -> Planner:
    """The process-wide planner the ops share (plan cache + table LRU)."""
    global _planner
    with _planner_lock:
        if _planner is None:
            _planner = Planner()
        return _planner


def _require_cuda(*ts):
    for t in ts:
        if t is not None and t.device.type != "cuda":
            raise RuntimeError("ftb ops run on the sm_100a executor only: inputs must be CUDA tensors "
                               f"(got {t.device})")


def _tma_ready(t: torch.Tensor) -> torch.Tensor:
    """A view with a contiguous last dim, row/batch strides that are multiples
    of 8 elements and a 16-byte aligned base (copying into a padded buffer
    only when needed)."""
    ok = t.stride(-1) == 1 and t.data_ptr() % 16 == 0 and all(s % 8 == 0 for s in t.stride()[:-1])
    if ok:
        return t
    cols = t.shape[-1]
    buf = t.new_zeros(*t.shape[:-1], (cols + 7) // 8 * 8 or 8)
    buf[..., :cols] = t
    return buf[..., :cols]


def _out_dtype(A: torch.Tensor) -> torch.dtype:
    return torch.float32 if A.dtype == torch.float32 else torch.bfloat16


@torch.library.custom_op("ftb::dense", mutates_args=())
def dense(A: torch.Tensor, B: torch.Tensor, b_layout: str = "nk", bias: Optional[torch.Tensor] = None,
          activation: str = "none") -> torch.Tensor:
    """act(A @ B + bias): A [M, K]; B [K, N] ("kn") or [N, K] ("nk", nn.Linear
    weight); bias [N] (bf16/fp32); activation "none" or "gelu" (erf form)."""
    _require_cuda(A, B, bias)
    act = None if activation == "none" else activation
    return planner().dense(_tma_ready(A), _tma_ready(B), b_layout=b_layout, bias=bias, activation=act)


@dense.register_fake
def _dense_fake(A, B, b_layout="nk", bias=None, activation="none"):
    N = B.shape[0] if b_layout == "nk" else B.shape[1]
    return A.new_empty((A.shape[0], N), dtype=_out_dtype(A))


@torch.library.custom_op("ftb::bmm", mutates_args=())
def bmm(A: torch.Tensor, B: torch.Tensor, b_layout: str = "kn", dynamic: str = "ij") -> torch.Tensor:
    """A [b, M, K] @ B ([b, K, N] "kn" or [b, N, K] "nk"); `dynamic` names the
    axes bound per call (attention scores "ij", context "ik")."""
    _require_cuda(A, B)
    return planner().bmm(_tma_ready(A), _tma_ready(B), b_layout=b_layout, dynamic=tuple(dynamic))


@bmm.register_fake
def _bmm_fake(A, B, b_layout="kn", dynamic="ij"):
    N = B.shape[1] if b_layout == "nk" else B.shape[2]
    return A.new_empty((A.shape[0], A.shape[1], N), dtype=torch.bfloat16)


def _shape_of(A, B, layout):
    if A.dim() == 2:
        N = B.shape[0] if layout == "nk" else B.shape[1]
        return (A.shape[0], N)
    N = B.shape[1] if layout == "nk" else B.shape[2]
    return (A.shape[0], A.shape[1], N)


@torch.library.custom_op("ftb::execute_table", mutates_args=())
def execute_table(As: List[torch.Tensor], Bs: List[torch.Tensor], b_layouts: str) -> List[torch.Tensor]:
    """Many Dense ([M, K]) and BatchMatmul ([b, M, K]) problems, each planned
    on its own, executed as ONE persistent launch (the grouped tile-schedule
    table); `b_layouts` is one "kn"/"nk" per problem, comma-separated. For
    repeated steps over the same buffers, ShapeSet / Executable amortise the
    table build; this op builds it per call."""
    b_layouts = b_layouts.split(",")
    if not (len(As) == len(Bs) == len(b_layouts)):
        raise ValueError("execute_table needs one B and one layout per A")
    _require_cuda(*As, *Bs)
    dtypes = {a.dtype for a in As} | {b.dtype for b in Bs}
    if len(dtypes) != 1:
        raise ValueError("one table shares one input dtype (bf16: tcgen05 kernel, fp32: FFMA validation kernel)")
    from .runtime import _ffma_planner

    pl = _ffma_planner() if dtypes == {torch.float32} else planner()
    As = [_tma_ready(a) for a in As]
    Bs = [_tma_ready(b) for b in Bs]
    insts, outs, descs = [], [], []
    for A, B, lay in zip(As, Bs, b_layouts):
        shape = _shape_of(A, B, lay)
        if A.dim() == 2:
            insts.append(dense_instance(A.shape[0], shape[1], A.shape[1], elem_bytes=4 if A.dtype == torch.float32 else 2))
        else:
            insts.append(bmm_instance(A.shape[0], A.shape[1], shape[2], A.shape[2]))
        outs.append(torch.empty(shape, dtype=_out_dtype(A), device=A.device))
        descs.append(gemm_desc(A, B, outs[-1], lay))
    recs = pl.plan(insts)
    ex = Executable(descs, [r.program for r in recs])
    ex.launch(torch.cuda.current_stream(As[0].device))
    ex.close()  # freed in stream order after the launch: no host or device sync
    return outs


@execute_table.register_fake
def _execute_table_fake(As, Bs, b_layouts):
    return [A.new_empty(_shape_of(A, B, lay), dtype=_out_dtype(A)) for A, B, lay in zip(As, Bs, b_layouts.split(","))]
