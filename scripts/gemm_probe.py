"""Main-loop probe: big square GEMMs with hand-made plans, single vs CTA-pair."""
import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct

def run(M, N, K, ti, tj, layout="nk", reps=10):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = (torch.rand(M, K, device="cuda", generator=g) - 0.5).bfloat16()
    B = (torch.rand(N, K, device="cuda", generator=g) - 0.5).bfloat16() if layout == "nk" else (torch.rand(K, N, device="cuda", generator=g) - 0.5).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    prog = program_struct(2, 0, [((1, 1), (ti, tj, 64), M // ti)])
    ex = Executable([gemm_desc(A, B, C, layout, orientation=0)], [prog], (A, B, C))
    for _ in range(3): ex.launch()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(reps): ex.launch(s)
    with torch.cuda.stream(s):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s); gr.replay(); e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    ref = (A.float() @ (B.float().t() if layout == "nk" else B.float()))
    err = ((C.float() - ref).abs().max() / ref.abs().max()).item()
    cfg = ex.config()
    print(f"M{M} N{N} K{K} tile {ti}x{tj} {layout} pair={os.environ.get('FTB_PAIR','1')}: {t*1e6:8.1f} us {2*M*N*K/t/1e12:7.1f} TF/s err {err:.1e} singles {cfg['n_singles']} pairs {cfg['n_pairs']} cfg1 {cfg['single']} cfg2 {cfg['pair']}", flush=True)
    # cuBLAS reference
    Bt = B.t() if layout == "nk" else B
    for _ in range(3): torch.matmul(A, Bt)
    torch.cuda.synchronize()
    e0.record(); 
    for _ in range(reps): torch.matmul(A, Bt)
    e1.record(); torch.cuda.synchronize()
    tc = e0.elapsed_time(e1) / reps * 1e-3
    print(f"   cuBLAS {tc*1e6:8.1f} us {2*M*N*K/tc/1e12:7.1f} TF/s")

for (M, N, K, ti, tj) in [(8192, 8192, 8192, 128, 256), (8192, 8192, 8192, 256, 256), (4096, 4096, 4096, 256, 256), (2048, 2304, 768, 256, 128), (4096, 3072, 768, 256, 256)]:
    run(M, N, K, ti, tj)
