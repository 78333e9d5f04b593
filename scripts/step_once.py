"""Launch the grouped C1 step table a few times (for ncu --set full captures):
  ncu --set full -k regex:ftb_tc -s 2 -c 1 -o OUT python scripts/step_once.py"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2407_21418_b200.runtime import Planner  # noqa: E402
from paper_2407_21418_b200.shapeset import ShapeSet  # noqa: E402
from paper_2407_21418_b200.workloads import c1_shapes  # noqa: E402

ss = ShapeSet(c1_shapes(24, 0), Planner(), device="cuda:0")
for _ in range(4):
    ss.launch()
torch.cuda.synchronize()
print("step launched", ss.exe.info.n_work, "items")
