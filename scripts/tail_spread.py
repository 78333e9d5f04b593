"""Tail imbalance of the grouped C1 step: per CTA, when its producer picks
its first item and when its last epilogue retires (device globaltimer, the
trace's item events; the last traced item of a CTA may not be its last item,
so the end is read from a dedicated per-CTA end stamp: the maximum of all
release events). Reports the spread of CTA end times. Needs the trace build
(the stamps are compiled out of the release kernel):
  make -C paper_2407_21418_b200/csrc trace (libftb_trace.so)."""
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ex.launch(); e1.record(); torch.cuda.synchronize()
print(f"step {e0.elapsed_time(e1)*1e3:.1f} us, items {ex.info.n_work}, ctas {ex.info.n_ctas}")
ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
ex.read_trace()
sp = ex.trace_span.astype(np.int64)[: ex.info.n_ctas]
t0 = sp[:, 0].min()
st, en = (sp[:, 0] - t0) / 1e3, (sp[:, 1] - t0) / 1e3
print(f"CTA start spread {st.min():.2f}..{st.max():.2f} us")
print(f"CTA end: min {en.min():.1f} p10 {np.percentile(en, 10):.1f} p50 {np.median(en):.1f} p90 {np.percentile(en, 90):.1f} max {en.max():.1f} us")
print(f"idle SM-time in the tail: {(en.max() - en).mean():.1f} us per CTA = {100 * (en.max() - en).mean() / en.max():.1f} % of the step")
