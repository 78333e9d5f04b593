"""Per-shape probe over C1's canonical shapes: planner plan (single / pair
kernels), a hand 'big tile' plan, and cuBLAS/torch.bmm for reference."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.workloads import bert_layer_shapes, CANONICAL_T

P = 1621.8e12
def timeit(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn()
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us

planner = Planner()
only = os.environ.get("ONLY")
for T in CANONICAL_T:
    for sh in bert_layer_shapes(T):
        if only and sh.kind != only: continue
        rec = planner.plan([sh.instance()])[0]
        g = torch.Generator(device="cuda").manual_seed(0)
        if sh.kind == "dense":
            A = (torch.rand(sh.M, sh.K, device="cuda", generator=g) - .5).bfloat16()
            B = (torch.rand(sh.N, sh.K, device="cuda", generator=g) - .5).bfloat16()
            C = torch.empty(sh.M, sh.N, device="cuda", dtype=torch.bfloat16)
            ref = lambda: torch.matmul(A, B.t())
        else:
            A = (torch.rand(sh.batch, sh.M, sh.K, device="cuda", generator=g) - .5).bfloat16()
            if sh.b_layout == "nk":
                B = (torch.rand(sh.batch, sh.N, sh.K, device="cuda", generator=g) - .5).bfloat16()
                ref = lambda: torch.bmm(A, B.transpose(1, 2))
            else:
                B = (torch.rand(sh.batch, sh.K, sh.N, device="cuda", generator=g) - .5).bfloat16()
                ref = lambda: torch.bmm(A, B)
            C = torch.empty(sh.batch, sh.M, sh.N, device="cuda", dtype=torch.bfloat16)
            if sh.K % 8 or sh.N % 8:
                continue
        res = {}
        for pair in ("0", "1"):
            os.environ["FTB_PAIR"] = pair
            ex = Executable([gemm_desc(A, B, C, sh.b_layout)], [rec.program], (A, B, C))
            res["p" + pair] = timeit(lambda: ex.launch(torch.cuda.current_stream()))
            ex.close()
        if sh.kind == "dense":
            tiles = [(128, 256), (256, 256), (256, 128)]
            for (ti, tj) in tiles:
                if sh.M % ti: continue
                prog = program_struct(2, 0, [((1, 1), (ti, tj, 64), sh.M // ti)])
                for pair in ("0", "1"):
                    os.environ["FTB_PAIR"] = pair
                    ex = Executable([gemm_desc(A, B, C, sh.b_layout, orientation=0)], [prog], (A, B, C))
                    res[f"{ti}x{tj}p{pair}"] = timeit(lambda: ex.launch(torch.cuda.current_stream()))
                    ex.close()
        tr = timeit(ref)
        roof = sh.t_roof(P) * 1e6
        plan = [(p['smem'], p['count']) for p in rec.describe()['parts']]
        print(f"{sh.name:8s} b{sh.batch:4d} M{sh.M:5d} N{sh.N:5d} K{sh.K:5d} roof {roof:7.2f}us torch {tr:7.2f} | " +
              " ".join(f"{k}={v:.2f}" for k, v in res.items()) + f" | plan {plan}", flush=True)
