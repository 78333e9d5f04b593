"""With a -DFTB_PROD_PROFILE build: producer clocks per K block spent waiting
for a free ring slot vs issuing, over the whole C1 table."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200 import _lib
_lib.LIB_PATH = __import__("pathlib").Path(sys.argv[1]).resolve()
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import c1_shapes
ops = os.environ.get("OPS", "dense")
shapes = [s for s in c1_shapes(24, 0) if ops == "all" or s.kind == ops]
ss = ShapeSet(shapes, Planner(), device="cuda:0")
ex = ss.exe
for _ in range(3): ex.launch()
ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
tr, kb = ex.read_trace()
raw = tr.reshape(tr.shape[0], -1)[:, :12].astype(np.float64)
wait, issue, item, nkb, nitems, total, m_te, m_full, m_issue, m_tot, e_wait, e_tot = raw.T
print(f"{ops}: per K block: wait {np.mean(wait/nkb):.0f} clk, issue {np.mean(issue/nkb):.0f} clk; "
      f"items/CTA {nitems.mean():.0f}, kb/CTA {nkb.mean():.0f}, total {total.mean():.0f} clk; "
      f"outside K loops {np.mean(total-item):.0f} clk ({np.mean((total-item)/nitems):.0f}/item)")
print(f"MMA warp: waiting TMEM {m_te.mean():.0f} clk, waiting data {m_full.mean():.0f}, issuing {m_issue.mean():.0f} of {m_tot.mean():.0f}; "
      f"epilogue warp2: waiting accumulators {e_wait.mean():.0f} of {e_tot.mean():.0f} clk")
print(f"per-CTA producer span: mean {total.mean():.0f} max {total.max():.0f} min {total.min():.0f} clk (max/mean {total.max()/total.mean():.3f}); epilogue span max/mean {e_tot.max()/e_tot.mean():.3f}")
