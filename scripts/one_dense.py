"""Run one Dense (env: M, N, K, LAYOUT, ORIENT) through the planner and executor; check vs float64."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner, dense_instance
M, N, K = (int(os.environ.get(k, d)) for k, d in (("M", 130), ("N", 1000), ("K", 256)))
lay, orient = os.environ.get("LAYOUT", "nk"), int(os.environ.get("ORIENT", "1"))
pad = lambda n: (n + 7) // 8 * 8  # noqa: E731
A = torch.randn(M, pad(K), device="cuda").bfloat16()[:, :K]
B = (torch.randn(K, pad(N), device="cuda").bfloat16()[:, :N] if lay == "kn"
     else torch.randn(N, pad(K), device="cuda").bfloat16()[:, :K])
Cb = torch.full((M, pad(N)), float("nan"), device="cuda").bfloat16()
C = Cb[:, :N]
rec = Planner().plan([dense_instance(M, N, K)])[0]
ex = Executable([gemm_desc(A, B, C, lay, orientation=orient)], [rec.program], (A, B, Cb))
print(rec.describe()["parts"], rec.describe()["tau"], ex.info.n_work, ex.info.n_ctas, ex.config()["single"], flush=True)
ex.launch(); torch.cuda.synchronize()
ref = A.double() @ (B.double() if lay == "kn" else B.double().t())
print("rel err", ((C.double() - ref).abs().max() / ref.abs().max()).item(), "pad untouched", torch.isnan(Cb[:, N:].float()).all().item())
