"""A shape set bound to device buffers and lowered to ONE tile-schedule table
(one persistent launch executes every shape), plus pinned host mirrors for
end-to-end runs. Used by bench.py, smoke() and the GPU tests."""

from __future__ import annotations

import time
from dataclasses import dataclass, field

from .execute import Executable, gemm_desc
from .runtime import Planner
from .workloads import Shape


def _round8(x: int) -> int:
    return (x + 7) // 8 * 8


@dataclass
class Bound:
    shape: Shape
    A: object          # device views passed to the executor
    B: object
    C: object
    A_store: object    # owning tensors (padded leading dims)
    C_store: object
    inputs: list = field(default_factory=list)   # per-step activations (H2D in e2e)


class ShapeSet:
    def __init__(self, shapes: list[Shape], planner: Planner | None = None, device="cuda", seed: int = 0,
                 pinned: bool = False):
        import torch

        self.shapes = shapes
        self.planner = planner or Planner()
        t0 = time.perf_counter()
        self.records = self.planner.plan([s.instance() for s in shapes])
        self.tuning_s = time.perf_counter() - t0
        self.device = torch.device(device)
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        dt = torch.bfloat16 if shapes[0].in_bytes == 2 else torch.float32

        def rnd(*shape):
            return (torch.rand(*shape, generator=g, device=self.device, dtype=torch.float32) * 2 - 1).to(dt)

        weights: dict = {}
        self.bound: list[Bound] = []
        for s in shapes:
            if s.kind == "dense":
                A = rnd(s.M, s.K)
                key = (s.name, s.N, s.K)
                if key not in weights:
                    weights[key] = rnd(s.N, s.K) if s.b_layout == "nk" else rnd(s.K, s.N)
                B = weights[key]
                C = torch.empty(s.M, s.N, dtype=dt, device=self.device)
                self.bound.append(Bound(s, A, B, C, A, C, [A]))
            else:
                b, T = s.batch, s.M
                if s.name == "scores":  # Q [b,T,64] @ K^T, K given as [b,T,64] ("nk")
                    A = rnd(b, s.M, s.K)
                    B = rnd(b, s.N, s.K)
                    Cs = torch.empty(b, s.M, _round8(s.N), dtype=dt, device=self.device)
                    C = Cs[:, :, : s.N]
                    self.bound.append(Bound(s, A, B, C, A, Cs, [A, B]))
                else:  # context: P [b,T,T] (row stride padded to 8) @ V [b,T,64] ("kn")
                    As = rnd(b, s.M, _round8(s.K))
                    A = As[:, :, : s.K]
                    B = rnd(b, s.K, s.N)
                    C = torch.empty(b, s.M, s.N, dtype=dt, device=self.device)
                    self.bound.append(Bound(s, A, B, C, As, C, [As, B]))
        self.weights = weights
        descs = [gemm_desc(x.A, x.B, x.C, x.shape.b_layout) for x in self.bound]
        keep = [t for x in self.bound for t in (x.A_store, x.B, x.C_store)]
        self.exe = Executable(descs, [r.program for r in self.records], keep)
        self.host_in = self.host_out = None
        if pinned:
            self.make_host_mirrors()

    # ------------------------------------------------------------------ e2e
    def make_host_mirrors(self):
        self.host_in = [[t.cpu().pin_memory() for t in x.inputs] for x in self.bound]
        self.host_out = [x.C_store.cpu().pin_memory() for x in self.bound]
        self.h2d_bytes = sum(t.numel() * t.element_size() for xs in self.host_in for t in xs)
        self.d2h_bytes = sum(t.numel() * t.element_size() for t in self.host_out)

    def step_e2e(self, stream=None):
        """Pinned host inputs -> device, one launch, outputs -> pinned host."""
        for x, hs in zip(self.bound, self.host_in):
            for d, h in zip(x.inputs, hs):
                d.copy_(h, non_blocking=True)
        self.exe.launch(stream)
        for x, h in zip(self.bound, self.host_out):
            h.copy_(x.C_store, non_blocking=True)

    def launch(self, stream=None):
        self.exe.launch(stream)

    # ------------------------------------------------------------------ stats
    @property
    def true_flops(self) -> int:
        return sum(s.flops for s in self.shapes)

    @property
    def alg_bytes(self) -> int:
        return sum(s.bytes for s in self.shapes)

    def padding_ratio(self) -> float:
        return self.exe.info.padding_ratio

    def reference_outputs(self, idx: int):
        """fp64 torch result of shape idx (for numerics checks on device)."""
        x = self.bound[idx]
        Bm = x.B.double()
        if x.shape.b_layout == "nk":
            Bm = Bm.transpose(-1, -2)
        return x.A.double() @ Bm
