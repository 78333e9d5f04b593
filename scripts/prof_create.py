import os, sys, time
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import c1_shapes
from paper_2407_21418_b200.execute import Executable, gemm_desc
sh = c1_shapes(24, 0)
pl = Planner()
ss = ShapeSet(sh, pl, device="cuda:0")
descs = [gemm_desc(x.A, x.B, x.C, x.shape.b_layout) for x in ss.bound]
for _ in range(3):
    t = time.perf_counter(); e = Executable(descs, [r.program for r in ss.records]); print("create total", (time.perf_counter() - t) * 1e3, "ms", flush=True)
