"""The C1 step as 192 cuBLAS calls (torch.matmul / torch.bmm) captured in one
CUDA graph — context for bench.py's grouped single-launch step."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.workloads import c1_shapes
shapes = c1_shapes(24, 0)
g = torch.Generator(device="cuda").manual_seed(0)
ops = []
for s in shapes:
    if s.kind == "dense":
        A = (torch.rand(s.M, s.K, device="cuda", generator=g) - .5).bfloat16()
        B = (torch.rand(s.N, s.K, device="cuda", generator=g) - .5).bfloat16()
        C = torch.empty(s.M, s.N, device="cuda", dtype=torch.bfloat16)
        ops.append(lambda A=A, B=B, C=C: torch.matmul(A, B.t(), out=C))
    else:
        A = (torch.rand(s.batch, s.M, s.K, device="cuda", generator=g) - .5).bfloat16()
        if s.b_layout == "nk":
            B = (torch.rand(s.batch, s.N, s.K, device="cuda", generator=g) - .5).bfloat16()
            C = torch.empty(s.batch, s.M, s.N, device="cuda", dtype=torch.bfloat16)
            ops.append(lambda A=A, B=B, C=C: torch.bmm(A, B.transpose(1, 2), out=C))
        else:
            B = (torch.rand(s.batch, s.K, s.N, device="cuda", generator=g) - .5).bfloat16()
            C = torch.empty(s.batch, s.M, s.N, device="cuda", dtype=torch.bfloat16)
            ops.append(lambda A=A, B=B, C=C: torch.bmm(A, B, out=C))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for op in ops: op()
torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=st):
    for op in ops: op()
for _ in range(5):
    with torch.cuda.stream(st): gr.replay()
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st); gr.replay(); e1.record(st)
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
fl = sum(s.flops for s in shapes)
print(f"cuBLAS C1 step (192 calls in one graph): {best:.4f} ms, {fl / best / 1e9:.1f} TF/s")
