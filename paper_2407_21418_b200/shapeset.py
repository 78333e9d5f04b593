"""A shape set bound to device buffers and lowered to ONE tile-schedule table
(one persistent launch executes every shape), plus pinned host mirrors for
end-to-end runs. Used by bench.py, smoke() and the GPU tests."""

from __future__ import annotations

import time
import zlib
from dataclasses import dataclass, field

from .execute import Executable, gemm_desc
from .runtime import Planner
from .workloads import Shape


def _round8(x: int) -> int:
    return (x + 7) // 8 * 8


def _arena(shapes, dtype, device):
    """One flat device allocation carved into views (128-B aligned)."""
    import math

    import torch

    esz = torch.tensor([], dtype=dtype).element_size()
    align = 128 // esz
    offs, n = [], 0
    for sh in shapes:
        offs.append(n)
        n += (math.prod(sh) + align - 1) // align * align
    buf = torch.empty(max(n, align), dtype=dtype, device=device)
    views = [buf[o:o + math.prod(sh)].view(*sh) for o, sh in zip(offs, shapes)]
    return views, buf


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
                 pinned: bool = False, seeds: list[int] | None = None, records=None):
        """``seeds``: one seed per shape — its activations are drawn from it and
        every weight from a hash of its (name, N, K, layout) key, so a shape's
        data does not depend on which other shapes share the set (the sharded
        C4 sweep checks per-shape checksums across partitions). ``records``:
        plans already made (skips planning)."""
        import torch

        self.shapes = shapes
        self.planner = planner or Planner()
        t0 = time.perf_counter()
        self.records = records if records is not None else self.planner.plan([s.instance() for s in shapes])
        self.tuning_s = time.perf_counter() - t0
        self.device = torch.device(device)
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        dt = torch.bfloat16 if shapes[0].in_bytes == 2 else torch.float32

        def rnd(*shape):
            return (torch.rand(*shape, generator=g, device=self.device, dtype=torch.float32) * 2 - 1).to(dt)

        weights: dict = {}
        self.bound: list[Bound] = []
        # Activations and outputs live in two contiguous arenas (views at
        # 128-B aligned offsets, as TMA needs), so an end-to-end step moves
        # its inputs and its outputs with one copy per direction.
        in_sizes, out_sizes = [], []
        for s in shapes:
            if s.kind == "dense":
                in_sizes.append([(s.M, s.K)])
                out_sizes.append((s.M, s.N))
            elif s.name == "scores":
                in_sizes.append([(s.batch, s.M, s.K), (s.batch, s.N, s.K)])
                out_sizes.append((s.batch, s.M, _round8(s.N)))
            else:
                in_sizes.append([(s.batch, s.M, _round8(s.K)), (s.batch, s.K, s.N)])
                out_sizes.append((s.batch, s.M, s.N))
        self._in_sizes, self._out_sizes, self._dt = in_sizes, out_sizes, dt
        in_views, self.in_arena = _arena([sh for xs in in_sizes for sh in xs], dt, self.device)
        out_views, self.out_arena = _arena(out_sizes, dt, self.device)
        if seeds is None:
            self.in_arena.copy_(rnd(self.in_arena.numel()))
        else:
            off = 0
            for sd, sizes in zip(seeds, in_sizes):
                for sh_ in sizes:
                    v = in_views[off]
                    off += 1
                    gs = torch.Generator(device=self.device)
                    gs.manual_seed(int(sd))
                    v.copy_((torch.rand(v.numel(), generator=gs, device=self.device) * 2 - 1).to(dt).view_as(v))

        def weight(key, *shape):
            if seeds is None:
                return rnd(*shape)
            gw = torch.Generator(device=self.device)
            gw.manual_seed(zlib.crc32(repr(key).encode()))
            return (torch.rand(*shape, generator=gw, device=self.device, dtype=torch.float32) * 2 - 1).to(dt)

        k = 0
        for s, oc in zip(shapes, out_views):
            if s.kind == "dense":
                A = in_views[k]
                k += 1
                key = (s.name, s.N, s.K, s.b_layout)
                if key not in weights:
                    weights[key] = weight(key, s.N, s.K) if s.b_layout == "nk" else weight(key, s.K, s.N)
                B = weights[key]
                self.bound.append(Bound(s, A, B, oc, A, oc, [A]))
            elif s.name == "scores":  # Q [b,T,64] @ K^T, K given as [b,T,64] ("nk")
                A, B = in_views[k], in_views[k + 1]
                k += 2
                self.bound.append(Bound(s, A, B, oc[:, :, : s.N], A, oc, [A, B]))
            else:  # context: P [b,T,T] (row stride padded to 8) @ V [b,T,64] ("kn")
                As, B = in_views[k], in_views[k + 1]
                k += 2
                self.bound.append(Bound(s, As[:, :, : s.K], B, oc, As, oc, [As, B]))
        self.weights = weights
        descs = [gemm_desc(x.A, x.B, x.C, x.shape.b_layout) for x in self.bound]
        keep = [self.in_arena, self.out_arena, *weights.values()]
        self.exe = Executable(descs, [r.program for r in self.records], keep)
        self.host_in = self.host_out = None
        if pinned:
            self.make_host_mirrors()

    # ------------------------------------------------------------------ e2e
    def make_host_mirrors(self):
        """Pinned host copies of the input and output arenas (one transfer per
        direction and step)."""
        self.host_in_arena = self.in_arena.cpu().pin_memory()
        self.host_out_arena = self.out_arena.cpu().pin_memory()
        self.host_in = True
        self.h2d_bytes = self.in_arena.numel() * self.in_arena.element_size()
        self.d2h_bytes = self.out_arena.numel() * self.out_arena.element_size()

    def _make_twin(self):
        """A second device buffer set (and its own lowered table: TMA
        descriptors embed addresses) so step k+1's inputs can stream in while
        step k computes and step k-1's outputs stream out."""
        in_views, in_arena = _arena([sh for xs in self._in_sizes for sh in xs], self._dt, self.device)
        out_views, out_arena = _arena(self._out_sizes, self._dt, self.device)
        twin, k = [], 0
        for x, oc in zip(self.bound, out_views):
            s = x.shape
            if s.kind == "dense":
                A = in_views[k]
                k += 1
                twin.append(Bound(s, A, x.B, oc, A, oc, [A]))
            elif s.name == "scores":
                A, B = in_views[k], in_views[k + 1]
                k += 2
                twin.append(Bound(s, A, B, oc[:, :, : s.N], A, oc, [A, B]))
            else:
                As, B = in_views[k], in_views[k + 1]
                k += 2
                twin.append(Bound(s, As[:, :, : s.K], B, oc, As, oc, [As, B]))
        descs = [gemm_desc(x.A, x.B, x.C, x.shape.b_layout) for x in twin]
        self.twin = twin
        self.twin_arenas = (in_arena, out_arena)
        self.exe_twin = Executable(descs, [r.program for r in self.records], (in_arena, out_arena, *self.weights.values()))

    def e2e_pipelined(self, steps: int, stream=None) -> float:
        """End-to-end steps through pinned host buffers with copies and compute
        overlapped across steps (H2D of step k+1 and D2H of step k-1 run on
        their own streams, full duplex, while step k computes). Every step
        still moves all of its inputs in and all of its outputs out. Returns
        ms per step (CUDA events, first H2D start to last D2H end)."""
        import torch

        if self.host_in is None:
            self.make_host_mirrors()
        if getattr(self, "exe_twin", None) is None:
            self._make_twin()
        comp = stream or torch.cuda.current_stream(self.device)
        h2d = torch.cuda.Stream(self.device)
        d2h = torch.cuda.Stream(self.device)
        sets = [(self.in_arena, self.out_arena, self.exe), (*self.twin_arenas, self.exe_twin)]
        ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731
        in_done, comp_done, out_done = [ev() for _ in range(steps)], [ev() for _ in range(steps)], [
            ev() for _ in range(steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(self.device)
        t0.record(h2d)
        for k in range(steps):
            in_arena, out_arena, exe = sets[k % 2]
            if k >= 2:
                h2d.wait_event(comp_done[k - 2])  # this buffer set's inputs are consumed
            with torch.cuda.stream(h2d):
                in_arena.copy_(self.host_in_arena, non_blocking=True)
                in_done[k].record(h2d)
            comp.wait_event(in_done[k])
            if k >= 2:
                comp.wait_event(out_done[k - 2])  # this buffer set's outputs were read back
            exe.launch(comp)
            comp_done[k].record(comp)
            d2h.wait_event(comp_done[k])
            with torch.cuda.stream(d2h):
                self.host_out_arena.copy_(out_arena, non_blocking=True)
                out_done[k].record(d2h)
        t1.record(d2h)
        torch.cuda.synchronize(self.device)
        return t0.elapsed_time(t1) / steps

    def step_e2e(self, stream=None):
        """Pinned host inputs -> device, one launch, outputs -> pinned host
        (serial, on one stream)."""
        self.in_arena.copy_(self.host_in_arena, non_blocking=True)
        self.exe.launch(stream)
        self.host_out_arena.copy_(self.out_arena, non_blocking=True)

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

    def checksums(self) -> list[dict]:
        """Per shape, on the device in float64: the sum of C and its
        size-independent expectation sum_k colsum(A)[k] * rowsum(B)[k]
        (= 1^T A B 1), plus sum |C| as the scale."""
        out = []
        for x in self.bound:
            Bkn = x.B.double().transpose(-1, -2) if x.shape.b_layout == "nk" else x.B.double()
            C = x.C.double()
            expect = (x.A.double().sum(-2) * Bkn.sum(-1)).sum()
            out.append({"sum": float(C.sum()), "expect": float(expect), "abs": float(C.abs().sum())})
        return out

    def reference_outputs(self, idx: int):
        """fp64 torch result of shape idx (for numerics checks on device)."""
        x = self.bound[idx]
        Bm = x.B.double()
        if x.shape.b_layout == "nk":
            Bm = Bm.transpose(-1, -2)
        return x.A.double() @ Bm
