"""Time the C1 dense step under alternative tilings (hand plans) to size the
gain available from the planner's B200 tile choice."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import c1_shapes

shapes = [s for s in c1_shapes(24, 0) if s.kind == "dense"]
ss = ShapeSet(shapes, Planner(), device="cuda:0")

def hand(s, variant):
    if variant == "128x256":
        if s.M <= 256:   # skinny: swap, lanes = j (128), cols = i (M)
            return program_struct(2, 1, [((1, 1), (s.M, 128, 64), s.N // 128)]), 1
        return program_struct(2, 1, [((1, 1), (128, 256, 64), s.N // 256)]), 0
    if variant == "256x256":
        if s.M <= 256:
            return program_struct(2, 1, [((1, 1), (s.M, 256, 64), s.N // 256)]), 1
        return program_struct(2, 1, [((1, 1), (256, 256, 64), s.N // 256)]), 0
    raise ValueError(variant)

def time_exe(ex, reps=20):
    for _ in range(5): ex.launch()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): ex.launch()
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best

flops = sum(s.flops for s in shapes)
t = time_exe(ss.exe)
print(f"planner plans: {t*1e3:.1f} us  {flops/t/1e9:.0f} TF/s  items {ss.exe.info.n_work}")
for v in ("128x256", "256x256"):
    descs, progs = [], []
    for x in ss.bound:
        p, o = hand(x.shape, v)
        descs.append(gemm_desc(x.A, x.B, x.C, x.shape.b_layout, o)); progs.append(p)
    ex = Executable(descs, progs)
    t = time_exe(ex)
    ref = x.A.float() @ x.B.float().t()
    err = ((x.C.float() - ref).abs().max() / ref.abs().max()).item()
    print(f"{v}: {t*1e3:.1f} us  {flops/t/1e9:.0f} TF/s  items {ex.info.n_work}  err(last) {err:.1e}  cfg {ex.config()['single']}")
