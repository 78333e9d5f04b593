"""Phase trace of the C1 step table (first 16 items of every CTA)."""
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
for _ in range(5): ex.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ex.launch(); e1.record(); torch.cuda.synchronize()
print(f"step {ops}: {e0.elapsed_time(e1)*1e3:.1f} us, items {ex.info.n_work}, cfg {ex.config()['single']}")
tab = ex.table()
ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
tr, kb = ex.read_trace(); tr = tr.astype(np.int64)
t0 = tr[tr > 0].min()
rel = np.where(tr > 0, tr - t0, -1) / 1e3
n = rel.shape[0]
for c in (0, 1, 70, 147):
    if c >= n: continue
    print(f"cta{c}:")
    for i in range(8):
        r = rel[c, i]
        w = c + i * n
        it = tab[w]
        print(f"  it{i} lanes {it[4]:3d} cols {it[5]:3d} nmma {it[6]:3d}  pick {r[0]:6.2f} k0land {r[2]:6.2f} commit {r[3]:6.2f} (mma {r[3]-r[2]:5.2f}) epi {r[4]:6.2f} rel {r[5]:6.2f} (epi {r[5]-r[4]:5.2f})")
ok = (rel[:, :, 5] >= 0)
mma = (rel[:, :, 3] - rel[:, :, 2])[ok]; epi = (rel[:, :, 5] - rel[:, :, 4])[ok]
gap = (rel[:, 1:, 2] - rel[:, :-1, 3])[ok[:, 1:]]
print(f"mean over traced items: mma {mma.mean():.2f} us, epi {epi.mean():.2f} us, gap (commit i -> k0land i+1) {gap.mean():.2f} us")
