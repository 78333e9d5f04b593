"""Per-shape time (20 launches in a CUDA graph) of the planner's plan vs
torch (cuBLAS) for C3 (Dense N=K=4096) and C2 (BERT-large attention BMM)."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.workloads import Shape

P = 1621.8e12
def timeit(fn, reps=20):
    torch.cuda.synchronize()  # launches of one table must not overlap (split-K workspace)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); g.replay(); e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best

pl = Planner()
shapes = [Shape("dense", "c3", 1, m, 4096, 4096, "nk") for m in (1, 16, 64, 127, 256, 1000, 2048, 4096, 8192)]
shapes += [Shape("bmm", "scores", 1024, t, t, 64, "nk", ("i", "j")) for t in (1, 64, 257, 512)]
shapes += [Shape("bmm", "context", 1024, t, 64, t, "kn", ("i", "k")) for t in (64, 256, 512)]
tot_ours = tot_torch = 0.0
for sh in shapes:
    rec = pl.plan([sh.instance()])[0]
    g = torch.Generator(device="cuda").manual_seed(0)
    if sh.kind == "dense":
        A = (torch.rand(sh.M, sh.K, device="cuda", generator=g) - .5).bfloat16()
        B = (torch.rand(sh.N, sh.K, device="cuda", generator=g) - .5).bfloat16()
        C = torch.empty(sh.M, sh.N, device="cuda", dtype=torch.bfloat16)
        ref = lambda: torch.matmul(A, B.t())
    else:
        kp = (sh.K + 7) // 8 * 8
        As = (torch.rand(sh.batch, sh.M, kp, device="cuda", generator=g) - .5).bfloat16()
        A = As[:, :, :sh.K]
        if sh.b_layout == "nk":
            B = (torch.rand(sh.batch, sh.N, sh.K, device="cuda", generator=g) - .5).bfloat16()
            ref = lambda: torch.bmm(A, B.transpose(1, 2))
        else:
            B = (torch.rand(sh.batch, sh.K, sh.N, device="cuda", generator=g) - .5).bfloat16()
            ref = lambda: torch.bmm(A, B)
        np_ = (sh.N + 7) // 8 * 8
        Cs = torch.empty(sh.batch, sh.M, np_, device="cuda", dtype=torch.bfloat16)
        C = Cs[:, :, :sh.N]
    ex = Executable([gemm_desc(A, B, C, sh.b_layout)], [rec.program])
    t = timeit(lambda: ex.launch(torch.cuda.current_stream()))
    tr = timeit(ref)
    tot_ours += t; tot_torch += tr
    roof = sh.t_roof(P) * 1e6
    d = rec.describe()
    print(f"{sh.name:7s} b{sh.batch:5d} M{sh.M:5d} N{sh.N:5d} K{sh.K:5d} roof {roof:8.2f}us ours {t:8.2f} ({roof/t:5.2f}) torch {tr:8.2f} ({roof/tr:5.2f}) items {ex.info.n_work:6d} plan {[(p['smem'], p['count']) for p in d['parts']]} stage {d['fallback_stage']}", flush=True)
print(f"sum ours {tot_ours:.1f} us, torch {tot_torch:.1f} us")
