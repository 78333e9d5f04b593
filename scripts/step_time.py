import os, sys, time
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import c1_shapes
ss = ShapeSet(c1_shapes(24, 0), Planner(), device="cuda:0")
s = torch.cuda.current_stream()
t_end = time.time() + 1.0
while time.time() < t_end:
    for _ in range(50): ss.launch(s)
    torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ss.launch(s); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"step {os.environ.get('TAG','')} median {ts[10]*1e3:.1f} us min {ts[0]*1e3:.1f} cfg {ss.exe.config()}")
