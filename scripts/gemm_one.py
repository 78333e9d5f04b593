import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct
M = N = K = int(os.environ.get("SZ", "8192")); ti, tj = int(os.environ.get("TI", "128")), 256
A = (torch.rand(M, K, device="cuda") - 0.5).bfloat16(); B = (torch.rand(N, K, device="cuda") - 0.5).bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ex = Executable([gemm_desc(A, B, C, "nk", orientation=0)], [program_struct(2, 0, [((1, 1), (ti, tj, 64), M // ti)])], (A, B, C))
for _ in range(3): ex.launch()
torch.cuda.synchronize(); print("done", ex.config())
