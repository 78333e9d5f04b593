"""Epilogue duration (trace events 4 -> 5) of a CTA's first item vs its later
items in the grouped C1 step: a cold instruction cache shows up as a slow
first epilogue."""
import os, sys
import os as _os
_os.environ.setdefault("FTB_LIB", "paper_2407_21418_b200/libftb_trace.so")  # phase traces need the trace build (make -C paper_2407_21418_b200/csrc trace)
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import c1_shapes
ops = os.environ.get("OPS", "dense")
shapes = [s for s in c1_shapes(24, 0) if ops == "all" or s.kind == ops]
ss = ShapeSet(shapes, Planner(), device="cuda:0")
ex = ss.exe
for _ in range(20): ex.launch()
torch.cuda.synchronize()
ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
tr, kb = ex.read_trace(); tr = tr.astype(np.int64)
n = ex.info.n_ctas
d = (tr[:n, :, 5] - tr[:n, :, 4]) / 1e3
ok = (tr[:n, :, 5] > 0) & (tr[:n, :, 4] > 0)
for i in range(8):
    v = d[:, i][ok[:, i]]
    print(f"item {i}: epilogue p50 {np.median(v):.2f} us  mean {v.mean():.2f}")
