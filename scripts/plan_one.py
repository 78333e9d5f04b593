"""Run one Dense shape with its planner plan (or a hand tile via TI/TJ) a few
times — a short command for ncu captures."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.workloads import Shape
M, N, K = (int(x) for x in os.environ.get("MNK", "768,768,3072").split(","))
A = (torch.rand(M, K, device="cuda") - 0.5).bfloat16(); B = (torch.rand(N, K, device="cuda") - 0.5).bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
if "TI" in os.environ:
    ti, tj = int(os.environ["TI"]), int(os.environ["TJ"])
    prog = program_struct(2, 0, [((1, 1), (ti, tj, 64), M // ti)])
else:
    prog = Planner().plan([Shape("dense", "x", 1, M, N, K, "nk").instance()])[0].program
ex = Executable([gemm_desc(A, B, C, "nk")], [prog], (A, B, C))
for _ in range(5): ex.launch()
torch.cuda.synchronize(); print("done", ex.config())
