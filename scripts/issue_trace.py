"""With a -DFTB_TRACE_ISSUE build: per K block, time spent issuing the TMA
loads (after the empty-slot wait) vs the wait itself."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200 import _lib
_lib.LIB_PATH = __import__("pathlib").Path(sys.argv[1]).resolve()
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import c1_shapes
ops = os.environ.get("OPS", "bmm")
shapes = [s for s in c1_shapes(24, 0) if ops == "all" or s.kind == ops]
ss = ShapeSet(shapes, Planner(), device="cuda:0")
ex = ss.exe
for _ in range(3): ex.launch()
ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
tr, kb = ex.read_trace(); kb = kb.astype(np.int64)
t0 = kb[kb > 0].min()
for c in (0, 70):
    pre = (kb[c, :24, 1] - t0) / 1e3; post = (kb[c, :24, 0] - t0) / 1e3
    print(f"cta{c} before-issue:", " ".join(f"{v:5.2f}" for v in pre))
    print(f"cta{c} after-issue :", " ".join(f"{v:5.2f}" for v in post))
d = (kb[:, :, 0] - kb[:, :, 1]); ok = (kb[:, :, 0] > 0) & (kb[:, :, 1] > 0)
print("mean issue duration us", d[ok].mean() / 1e3, " median", np.median(d[ok]) / 1e3)
