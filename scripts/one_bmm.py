"""Run one BMM (env: B, M, N, K, LAYOUT) through the planner and executor; check vs float64."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner, bmm_instance
b, M, N, K = (int(os.environ.get(k, d)) for k, d in (("B", 1), ("M", 228), ("N", 228), ("K", 64)))
lay = os.environ.get("LAYOUT", "kn")
pad = lambda n: (n + 7) // 8 * 8  # noqa: E731
A = torch.randn(b, M, pad(K), device="cuda").bfloat16()[:, :, :K]
Bt = (torch.randn(b, K, pad(N), device="cuda").bfloat16()[:, :, :N] if lay == "kn"
      else torch.randn(b, N, pad(K), device="cuda").bfloat16()[:, :, :K])
npad = (N + 7) // 8 * 8
C = torch.full((b, M, npad), float("nan"), device="cuda").bfloat16()[:, :, :N]
if os.environ.get("COMPACT"):  # C rows not padded to 16 B: the bulk row-store path
    C = torch.full((b, M, N), float("nan"), device="cuda").bfloat16()
rec = Planner().plan([bmm_instance(b, M, N, K)])[0]
ex = Executable([gemm_desc(A, Bt, C, lay)], [rec.program], (A, Bt, C))
print(rec.describe()["parts"], rec.describe()["tau"], ex.info.n_work, ex.info.n_ctas, ex.config()["single"], flush=True)
print(ex.table().tolist(), flush=True)
ex.launch(); torch.cuda.synchronize()
ref = A.double() @ (Bt.double() if lay == "kn" else Bt.double().transpose(1, 2))
print("rel err", ((C.double() - ref).abs().max() / ref.abs().max()).item())
