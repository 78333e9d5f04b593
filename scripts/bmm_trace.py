"""Phase trace of one attention BMM table (env B, T, KIND=scores|context):
is it epilogue bound? Prints the mean MMA span and epilogue span per item
and the per-item cadence (trace build)."""
import os as _os
_os.environ.setdefault("FTB_LIB", "paper_2407_21418_b200/libftb_trace.so")
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner, bmm_instance
b, T = int(os.environ.get("B", "1024")), int(os.environ.get("T", "512"))
kind = os.environ.get("KIND", "scores")
if kind == "scores":
    A = torch.randn(b, T, 64, device="cuda").bfloat16(); Bt = torch.randn(b, T, 64, device="cuda").bfloat16(); lay = "nk"
    C = torch.empty(b, T, T, device="cuda", dtype=torch.bfloat16); inst = bmm_instance(b, T, T, 64)
else:
    A = torch.randn(b, T, T, device="cuda").bfloat16(); Bt = torch.randn(b, T, 64, device="cuda").bfloat16(); lay = "kn"
    C = torch.empty(b, T, 64, device="cuda", dtype=torch.bfloat16); inst = bmm_instance(b, T, 64, T, ("i", "k"))
ex = Executable([gemm_desc(A, Bt, C, lay)], [Planner().plan([inst])[0].program], (A, Bt, C))
for _ in range(5): ex.launch()
torch.cuda.synchronize()
ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
tr, kb = ex.read_trace(); tr = tr.astype(np.int64)
n = ex.info.n_ctas
ok = (tr[:n, :, 5] > 0) & (tr[:n, :, 2] > 0)
mma = ((tr[:n, :, 3] - tr[:n, :, 2]) / 1e3)[ok]
epi = ((tr[:n, :, 5] - tr[:n, :, 4]) / 1e3)[ok]
cad = (np.diff(tr[:n, :, 0], axis=1) / 1e3)[ok[:, 1:]]
print(f"{kind} b{b} T{T}: items {ex.info.n_work} ctas {n} cfg {ex.config()['single']}")
print(f"  per item: MMA span {mma.mean():.2f} us, epilogue {epi.mean():.2f} us, producer pick cadence {cad.mean():.2f} us")
