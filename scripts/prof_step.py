"""clock64 role profile (libftb_prof.so) of the grouped C1 step: per-CTA
producer / MMA / epilogue busy and wait cycles, and the spread of CTA
finish times (static round-robin load balance).
  python scripts/prof_step.py"""
import os
import sys

os.environ.setdefault("FTB_LIB", "paper_2407_21418_b200/libftb_prof.so")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_21418_b200.runtime import Planner  # noqa: E402
from paper_2407_21418_b200.shapeset import ShapeSet  # noqa: E402
from paper_2407_21418_b200.workloads import c1_shapes  # noqa: E402

ss = ShapeSet(c1_shapes(24, 0), Planner(), device="cuda:0")
ex = ss.exe
ex.set_trace(True)
for _ in range(20):
    ex.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ex.launch()
e1.record()
torch.cuda.synchronize()
tr, _ = ex.read_trace()
n = ex.info.n_ctas
raw = tr.reshape(tr.shape[0], -1)[:n, :12].astype(np.float64)
p_wait, p_issue, p_item, nkb, nitems, p_total, m_te, m_full, m_issue, m_total, e_wait, e_total = raw.T
print(f"step {e0.elapsed_time(e1) * 1e3:.1f} us, ctas {n}, items/CTA {nitems.mean():.1f} (min {nitems.min():.0f} max {nitems.max():.0f}), "
      f"kb/CTA {nkb.mean():.0f} (min {nkb.min():.0f} max {nkb.max():.0f}) cfg {ex.config()['single']}")
for name, v in (("producer total", p_total), ("producer wait-slot", p_wait), ("producer issue", p_issue),
                ("mma total", m_total), ("mma wait-tmem", m_te), ("mma wait-data", m_full), ("mma issue", m_issue),
                ("epi total", e_total), ("epi wait-acc", e_wait)):
    print(f"  {name:20s} mean {v.mean():9.0f}  min {v.min():9.0f}  max {v.max():9.0f} clk")
print(f"  MMA issue per kb {np.mean(m_issue / np.maximum(nkb, 1)):.0f} clk; producer issue per kb {np.mean(p_issue / np.maximum(nkb, 1)):.0f} clk")
