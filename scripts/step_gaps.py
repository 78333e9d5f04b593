"""MMA idle gaps in the grouped C1 step, by item kind: for each traced item,
gap = (first K block of item i lands) - (item i-1 committed), i.e. time the
MMA warp waited for data. BMM (1-2 K blocks: MMA span < 1 us) vs Dense (>= 12 K blocks)."""
import sys
import os as _os
_os.environ.setdefault("FTB_LIB", "paper_2407_21418_b200/libftb_trace.so")  # phase traces need the trace build (make -C paper_2407_21418_b200/csrc trace)
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import c1_shapes
ss = ShapeSet(c1_shapes(24, 0), Planner(), device="cuda:0")
ex = ss.exe
for _ in range(20): ex.launch()
torch.cuda.synchronize()
ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
tr, kb = ex.read_trace(); tr = tr.astype(np.int64)
n = ex.info.n_ctas
gaps = {"dense": [], "bmm": []}
mma = {"dense": [], "bmm": []}
for c in range(n):
    for i in range(1, 16):
        if tr[c, i, 2] <= 0 or tr[c, i - 1, 3] <= 0 or tr[c, i, 3] <= 0:
            continue
        span = (tr[c, i, 3] - tr[c, i, 2]) / 1e3
        kind = "bmm" if span < 1.0 else "dense"  # 1-2 K blocks vs >= 12
        gaps[kind].append((tr[c, i, 2] - tr[c, i - 1, 3]) / 1e3)
        mma[kind].append((tr[c, i, 3] - tr[c, i, 2]) / 1e3)
for k in gaps:
    g = np.array(gaps[k]); m = np.array(mma[k])
    if len(g):
        print(f"{k:5s}: items {len(g)}  MMA wait before item (us) mean {g.mean():.3f} p50 {np.median(g):.3f} p90 {np.percentile(g, 90):.3f}"
              f"  | item MMA span mean {m.mean():.3f}")
