import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200 import _lib
_lib.LIB_PATH = __import__("pathlib").Path(sys.argv[1]).resolve()
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct
M, N, K = (int(x) for x in os.environ.get("MNK", "4096,3072,768").split(","))
A = (torch.rand(M, K, device="cuda") - 0.5).bfloat16(); B = (torch.rand(N, K, device="cuda") - 0.5).bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ex = Executable([gemm_desc(A, B, C, "nk", 0)], [program_struct(2, 0, [((1, 1), (256, int(os.environ.get("TJ", "256")), 64), M // 256)])], (A, B, C))
for _ in range(3): ex.launch()
ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
tr, kb = ex.read_trace()
raw = tr.reshape(tr.shape[0], -1)[:, :6].astype(np.float64)
wait, issue, item, nkb, nitems, total = raw.T
print(os.environ.get("FTB_PAIR"), ex.config()["n_pairs"], f"per K block: wait {np.mean(wait/nkb):.0f} clk, issue {np.mean(issue/nkb):.0f} clk; items/CTA {nitems.mean():.1f}, kb/CTA {nkb.mean():.0f}, total {total.mean():.0f} clk")
if os.environ.get("FTB_PAIR") == "1":
    for r in (0, 1):
        sel = slice(r, None, 2)
        print(f"  rank {r}: wait {np.mean(wait[sel]/nkb[sel]):.0f} issue {np.mean(issue[sel]/nkb[sel]):.0f} clk per K block")
