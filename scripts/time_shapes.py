"""us per launch (CUDA graph of 20, best of 3) for Dense shapes SHAPES="M N K;..." (nk)."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.calibrate import time_launches
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner, dense_instance
for spec in os.environ.get("SHAPES", "127 4096 4096;160 768 3072;768 768 3072").split(";"):
    M, N, K = map(int, spec.split())
    A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    orient = int(os.environ.get("ORIENT", "-1"))
    ex = Executable([gemm_desc(A, B, C, "nk", orientation=orient)], [Planner().plan([dense_instance(M, N, K)])[0].program],
                    (A, B, C))
    for _ in range(200): ex.launch()
    us = time_launches(lambda s: ex.launch(s), reps=20)
    ref = A.float() @ B.float().t()
    err = ((C.float() - ref).abs().max() / ref.abs().max()).item()
    print(f"M{M} N{N} K{K}: {us:.2f} us  ctas {ex.info.n_ctas}  err {err:.1e}", flush=True)
    ex.close()
