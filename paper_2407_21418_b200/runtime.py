"""Runtime front door: plan dynamic shapes with the C++ planner (cached) and
execute them with the sm_100a executor.

    pl = Planner()                          # B200 descriptor, tcgen05 mode
    C = pl.dense(A, W, b_layout="nk")       # plan (cached per shape) + one launch
    progs = pl.plan([dense_instance(M, 2304, 768) for M in Ms])   # batch tuning

The planner is the reference's analytic pipeline (compile stage + runtime
stage + SIA Top-1) run per shape in C++ on a host thread
pool; planning time is reported as "tuning seconds" and never lands inside a
timed kernel region. The plan cache is keyed by (descriptor, workload hash,
binding), the f-1 "persistent plan cache" of SURVEY.md §8.
"""

from __future__ import annotations

import ctypes as C
import functools
import json
import os
import threading
import time
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

from . import _lib
from .execute import Executable, gemm_desc
from .mktune import _native
from .mktune.filtering import FilterParams
from .mktune.hardware import HardwareDescriptor, b200_bf16, b200_ffma
from .mktune.scoring import SiaCoeffs
from .mktune.workload import WorkloadInstance, bmm_spec, dense_spec, workload_hash

CACHE_VERSION = 3


@functools.lru_cache(maxsize=4096)
def _dense_spec(N: int, K: int, hi: int, elem_bytes: int):
    return dense_spec(N, K, (1, hi), elem_bytes)


@functools.lru_cache(maxsize=4096)
def _bmm_spec(b: int, i, j, k, elem_bytes: int, name: str):
    return bmm_spec(b, i, j, k, elem_bytes=elem_bytes, name=name)


def spec_hash(spec) -> str:
    """workload_hash(spec), memoised on the (frozen) spec object: the runtime's
    plan-cache key is computed per call, and the canonical-JSON hash costs
    ~35 us (the specs of dense_instance / bmm_instance are memoised too, so a
    dynamic-shape step's cache hits cost microseconds, not ~85 us each)."""
    h = spec.__dict__.get("_ftb_hash")
    if h is None:
        h = workload_hash(spec)
        object.__setattr__(spec, "_ftb_hash", h)
    return h


def dense_instance(M: int, N: int, K: int, elem_bytes: int = 2, m_max: int = 8192) -> WorkloadInstance:
    return WorkloadInstance(_dense_spec(N, K, max(m_max, M), elem_bytes), {"i": M})


def bmm_instance(b: int, M: int, N: int, K: int, dynamic=("i", "j"), elem_bytes: int = 2,
                 t_max: int = 512) -> WorkloadInstance:
    """BatchMatmul instance; ``dynamic`` names the axes bound per call
    (scores: i, j = T; context: i, k = T)."""
    ext = {"i": M, "j": N, "k": K}
    hi = max(t_max, M, N, K)
    spec = _bmm_spec(b, *[((1, hi) if a in dynamic else ext[a]) for a in ("i", "j", "k")], elem_bytes,
                     "bmm-" + "".join(dynamic))
    return WorkloadInstance(spec, {a: ext[a] for a in dynamic})


@dataclass
class PlanRecord:
    program: _lib.Program
    tuning_s: float
    relaxation: str
    stage: int
    counts: dict

    def describe(self) -> dict:
        g = self.program
        parts = []
        for p in range(g.n_parts):
            parts.append({"smem": [int(g.smem[p][a]) for a in range(g.n_space + g.n_reduce)],
                          "reg": [int(g.reg[p][a]) for a in range(g.n_space)], "count": int(g.count[p])})
        return {"tau": int(g.tau), "parts": parts, "sia": float(g.sia), "relaxation": self.relaxation,
                "fallback_stage": self.stage, "tuning_s": self.tuning_s, "counts": self.counts}


def native_cover_program(inst: WorkloadInstance) -> _lib.Program:
    """Last rung of the runtime planner's fallback ladder (beyond the
    reference): an exact cover of the composition axis built directly from
    executor tiles, for shapes whose uKernel candidates admit no exact
    combination (e.g. a main-axis extent that is not a multiple of the
    64-element alignment; the reference raises EmptyResultError there,
    combine.py:183-188, and so does the mktune facade). BMM: tau = batch, one
    entry per tile. Dense: tau = i, 128-row tiles plus one ragged tile. Other
    space axes: uniform tiles (the executor cuts every rectangle into MMA
    items anyway); reduce tile 64; register tiles 1."""
    from .execute import program_struct

    spec = inst.spec
    space = list(spec.space_axes)
    ext = inst.extents
    if len(space) == 3:  # BMM: b, i, j
        tau = 0
        tiles = [1, min(ext[space[1]], 128), min(ext[space[2]], 256), 64]
        parts = [([1, 1, 1], tiles, ext[space[0]])]
    else:  # Dense: i, j
        tau = 0
        M = ext[space[0]]
        jt = min(ext[space[1]], 256)
        full, rem = divmod(M, 128)
        parts = []
        if full:
            parts.append(([1, 1], [128, jt, 64], full))
        if rem:
            parts.append(([1, 1], [rem, jt, 64], 1))
    return program_struct(len(space), tau, parts)


class Planner:
    """Thread-safe plan cache over the C++ planner. Shapes whose candidates
    admit no exact cover even after the C++ fallback ladder get
    `native_cover_program` (relaxation "native-cover", stage -1) unless
    ``native_cover`` is False (or FTB_NATIVE_COVER=0), in which case the
    reference's EmptyResultError is raised."""

    def __init__(self, hw: HardwareDescriptor | None = None, params: FilterParams | None = None,
                 coeffs: SiaCoeffs | None = None, threads: int = 0):
        self.hw = hw or b200_bf16(tcgen05=True)
        self.params = params or FilterParams.default()
        if coeffs is None and os.environ.get("FTB_SIA_COEFFS"):
            coeffs = SiaCoeffs(*(float(v) for v in os.environ["FTB_SIA_COEFFS"].split(",")))
        self.coeffs = coeffs or SiaCoeffs()
        self.threads = threads
        self.native_cover = os.environ.get("FTB_NATIVE_COVER", "1") != "0"
        # the whole descriptor (name + every field, tcgen05 ones included) keys the cache
        self._hw_key = json.dumps(self.hw.to_doc(), sort_keys=True)
        self._cache: dict[tuple, PlanRecord] = {}
        self._exe_cache: dict[tuple, Executable] = {}  # insertion-ordered LRU of lowered tables
        self._op_plans: dict[tuple, PlanRecord] = {}   # (op, extents, ...) -> plan: skips instance building on hits
        self.exe_cache_size = 32
        self._lock = threading.Lock()

    def _key(self, inst: WorkloadInstance) -> tuple:
        c = self.coeffs
        return (self._hw_key, (c.c0, c.c1, c.c2), spec_hash(inst.spec), inst.binding_key())

    def plan(self, instances: Sequence[WorkloadInstance]) -> list[PlanRecord]:
        """Top-1 program per instance (cached); misses are planned in one
        multi-threaded C++ call."""
        keys = [self._key(i) for i in instances]
        with self._lock:
            miss = [j for j, k in enumerate(keys) if k not in self._cache]
        if miss:
            uniq: dict[tuple, int] = {}
            for j in miss:
                uniq.setdefault(keys[j], j)
            todo = list(uniq.values())
            n = len(todo)
            insts = (_native.Inst * n)(*[_native.inst_struct(instances[j], self.params.major_axis) for j in todo])
            progs = (_lib.Program * n)()
            reps = (_native.Report * n)()
            stats = (C.c_int32 * n)()
            _lib.check(_native.lib().ftb_plan_batch(
                C.byref(_native.hw_struct(self.hw)), insts, n, C.byref(_native.params_struct(self.params)),
                C.byref(_native.coeffs_struct(self.coeffs)), self.threads, progs, reps, stats))
            for q, j in enumerate(todo):
                if stats[q] == _lib.FTB_EMPTY_RESULT and self.native_cover:
                    rec = PlanRecord(program=native_cover_program(instances[j]), tuning_s=reps[q].seconds,
                                     relaxation="native-cover", stage=-1, counts={})
                    with self._lock:
                        self._cache[keys[j]] = rec
                    continue
                if stats[q] != 0:
                    # re-plan alone to surface the exact error text / class
                    one = (_native.Inst * 1)(insts[q])
                    _lib.check(_native.lib().ftb_plan_batch(
                        C.byref(_native.hw_struct(self.hw)), one, 1, C.byref(_native.params_struct(self.params)),
                        C.byref(_native.coeffs_struct(self.coeffs)), 1, (_lib.Program * 1)(), None, None))
                r = reps[q]
                rec = PlanRecord(
                    program=_lib.Program.from_buffer_copy(progs[q]), tuning_s=r.seconds,
                    relaxation=_native.relaxation_name(r.relaxation, r.widen), stage=r.stage,
                    counts={"align": r.n_align, "cross": r.n_cross, "filter": r.n_filter, "final": r.n_final})
                with self._lock:
                    self._cache[keys[j]] = rec
        with self._lock:
            return [self._cache[k] for k in keys]

    # ---------------------------------------------------------------- ops

    def _launch(self, rec, A, B, out, b_layout, bias=None, activation=None, stream=None):
        """Launch one planned problem through a small cache of lowered tables.

        TMA descriptors embed buffer addresses, so the key holds each tensor's
        (address, shape, strides, dtype, device). The cache does NOT keep the
        tensors alive: a cached table is only ever launched again for tensors
        matching its key exactly — the same bytes it was built for — so a
        freed-and-reused address is harmless, and evicting a table never
        synchronises the device (exec.cu frees it in stream order after its
        last launch)."""
        key = tuple((t.data_ptr(), tuple(t.shape), tuple(t.stride()), t.dtype, t.device)
                    if t is not None else None for t in (A, B, out, bias)) + (b_layout, activation, id(rec))
        with self._lock:
            ex = self._exe_cache.pop(key, None)
        if ex is None:
            ex = Executable([gemm_desc(A, B, out, b_layout, bias=bias, activation=activation)], [rec.program],
                            (rec,))
        ex.launch(stream if stream is not None else _current_stream(A.device))
        with self._lock:
            self._exe_cache[key] = ex
            while len(self._exe_cache) > self.exe_cache_size:
                self._exe_cache.pop(next(iter(self._exe_cache)))
        return out

    def _memo_op(self, key, rec) -> None:
        """Bounded memo of the op entry points (the plan cache itself stays
        complete): a serving process with unbounded shape variety does not
        grow it without limit."""
        if len(self._op_plans) >= 65536:
            self._op_plans.clear()
        self._op_plans[key] = rec

    def dense(self, A, B, b_layout: str = "kn", out=None, stream=None, bias=None, activation=None):
        """C = act(A @ B + bias) (B as [K,N] for "kn", as nn.Linear weight [N,K]
        for "nk"); bias [N] and activation ("gelu") are fused into the epilogue."""
        import torch

        M, K = A.shape
        N = B.shape[1] if b_layout == "kn" else B.shape[0]
        fp32 = A.dtype == torch.float32
        rec = self._op_plans.get(("dense", M, N, K, fp32))
        if rec is None:
            inst = dense_instance(M, N, K, elem_bytes=4 if fp32 else 2)
            planner = self if (not fp32 or not self.hw.tcgen05_mode) else _ffma_planner()
            rec = planner.plan([inst])[0]
            self._memo_op(("dense", M, N, K, fp32), rec)
        if out is None:
            out = torch.empty(M, N, dtype=torch.float32 if fp32 else torch.bfloat16, device=A.device)
        return self._launch(rec, A, B, out, b_layout, bias, activation, stream)

    def bmm(self, A, B, b_layout: str = "kn", dynamic=("i", "j"), out=None, stream=None):
        import torch

        b, M, K = A.shape
        N = B.shape[2] if b_layout == "kn" else B.shape[1]
        key = ("bmm", b, M, N, K, tuple(dynamic))
        rec = self._op_plans.get(key)
        if rec is None:
            rec = self.plan([bmm_instance(b, M, N, K, dynamic)])[0]
            self._memo_op(key, rec)
        if out is None:
            out = torch.empty(b, M, N, dtype=torch.bfloat16, device=A.device)
        return self._launch(rec, A, B, out, b_layout, stream=stream)

    # ---------------------------------------------------------------- persistence

    def save(self, path: str | Path) -> None:
        """Write the plan cache (plan file: SPEC.md:412; versioned)."""
        with self._lock:
            rows = [{"key": list(k), **v.describe(), "n_space": v.program.n_space}
                    for k, v in self._cache.items()]
        Path(path).write_text(json.dumps({"version": CACHE_VERSION, "hw": self.hw.to_doc(), "plans": rows},
                                         sort_keys=True, indent=1) + "\n")

    def load(self, path: str | Path) -> int:
        doc = json.loads(Path(path).read_text())
        if doc.get("version") != CACHE_VERSION or doc.get("hw") != self.hw.to_doc():
            return 0
        from .execute import program_struct

        n = 0
        for row in doc["plans"]:
            parts = [(p["reg"], p["smem"], p["count"]) for p in row["parts"]]
            g = program_struct(row["n_space"], row["tau"], parts, row["sia"])
            with self._lock:
                key = tuple(tuple(x) if isinstance(x, list) else x for x in row["key"])
                self._cache[key] = PlanRecord(g, row["tuning_s"], row["relaxation"],
                                                            row["fallback_stage"], row["counts"])
            n += 1
        return n


def _current_stream(device):
    import torch

    return torch.cuda.current_stream(device)


_FFMA = None


def _ffma_planner() -> Planner:
    global _FFMA
    if _FFMA is None:
        _FFMA = Planner(hw=b200_ffma())
    return _FFMA


def timed_plan(planner: Planner, instances) -> tuple[list[PlanRecord], float]:
    t0 = time.perf_counter()
    recs = planner.plan(instances)
    return recs, time.perf_counter() - t0
