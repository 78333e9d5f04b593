"""One S^3 bf16 GEMM launch (env S, default 8192) for ncu captures."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner, dense_instance
S = int(os.environ.get("S", "8192"))
A = torch.randn(S, S, device="cuda").bfloat16(); B = torch.randn(S, S, device="cuda").bfloat16()
C = torch.empty(S, S, device="cuda", dtype=torch.bfloat16)
ex = Executable([gemm_desc(A, B, C, "nk")], [Planner().plan([dense_instance(S, S, S)])[0].program], (A, B, C))
for _ in range(3): ex.launch()
torch.cuda.synchronize()
if os.environ.get("CUBLAS"):
    for _ in range(3): torch.matmul(A, B.t(), out=C)
    torch.cuda.synchronize()
