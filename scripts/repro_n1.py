import sys, itertools
sys.path.insert(0, "/root/repo")
import torch, torch.nn.functional as F
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner, dense_instance
M, N, K = 2, 1, 256
for lay, orient, bias_on, act in itertools.product(["kn", "nk"], [0, 1], [False, True], [None, "gelu"]):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(K, 8, device="cuda").bfloat16()[:, :N] if lay == "kn" else torch.randn(N, K, device="cuda").bfloat16())
    Cb = torch.full((M, 16), float("nan"), device="cuda").bfloat16(); C = Cb[:, :N]
    bias = torch.randn(N, device="cuda").bfloat16() if bias_on else None
    rec = Planner().plan([dense_instance(M, N, K)])[0]
    ex = Executable([gemm_desc(A, B, C, lay, orientation=orient, bias=bias, activation=act)], [rec.program], (A, B, Cb, bias))
    ex.launch(); torch.cuda.synchronize()
    ref = A.double() @ (B.double() if lay == "kn" else B.double().t())
    if bias_on: ref = ref + bias.double()
    if act: ref = F.gelu(ref)
    err = ((C.double() - ref).abs().max() / ref.abs().max()).item()
    print(lay, orient, bias_on, act, f"err {err:.2e}", C.flatten().tolist(), ref.flatten().tolist(), flush=True)
