"""A/B timing of two builds of libftb.so on the same box, same process, same
buffers: python scripts/ab_test.py LIB_A LIB_B  (shapes: C1 canonical)."""
import ctypes as C
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200 import _lib
from paper_2407_21418_b200.execute import gemm_desc, program_struct
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.workloads import bert_layer_shapes, CANONICAL_T, Shape

libs = [C.CDLL(p) for p in sys.argv[1:]]
for L in libs:
    L.ftb_exec_create.restype = C.c_int32
    L.ftb_exec_launch.restype = C.c_int32

def timeit(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s); fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn(s)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); g.replay(); e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps * 1e3)
    return best

REPS = 20
def make_graph(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s); fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(REPS): fn(s)
    return (g, s)

def time_graph(gs):
    g, s = gs
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / REPS * 1e3

planner = Planner()
shapes = []
if os.environ.get("SHAPES") == "big":
    shapes = [(Shape("dense", "sq", 1, 4096, 4096, 4096, "nk"), (256, 256)), (Shape("dense", "sq", 1, 4096, 3072, 768, "nk"), (128, 256)),
              (Shape("dense", "sq", 1, 4096, 3072, 768, "nk"), (256, 256)), (Shape("dense", "sq", 1, 8192, 8192, 8192, "nk"), (256, 256))]
else:
    for T in CANONICAL_T[1::2]:
        for sh in bert_layer_shapes(T):
            shapes.append((sh, None))
for sh, tile in shapes:
    g = torch.Generator(device="cuda").manual_seed(0)
    if sh.kind == "dense":
        A = (torch.rand(sh.M, sh.K, device="cuda", generator=g) - .5).bfloat16()
        B = (torch.rand(sh.N, sh.K, device="cuda", generator=g) - .5).bfloat16()
        Cm = torch.empty(sh.M, sh.N, device="cuda", dtype=torch.bfloat16)
    else:
        if sh.K % 8 or sh.N % 8: continue
        A = (torch.rand(sh.batch, sh.M, sh.K, device="cuda", generator=g) - .5).bfloat16()
        B = (torch.rand(sh.batch, *((sh.N, sh.K) if sh.b_layout == "nk" else (sh.K, sh.N)), device="cuda", generator=g) - .5).bfloat16()
        Cm = torch.empty(sh.batch, sh.M, sh.N, device="cuda", dtype=torch.bfloat16)
    if tile:
        prog = program_struct(2, 0, [((1, 1), (tile[0], tile[1], 64), sh.M // tile[0])])
    else:
        prog = planner.plan([sh.instance()])[0].program
    d = (_lib.GemmDesc * 1)(gemm_desc(A, B, Cm, sh.b_layout))
    p = (_lib.Program * 1)(prog)
    graphs = []
    for pair in os.environ.get("PAIRS", "0,1").split(","):
        os.environ["FTB_PAIR"] = pair
        for L in libs:
            h = C.c_void_p()
            assert L.ftb_exec_create(d, p, 1, C.byref(h)) == 0
            graphs.append(make_graph(lambda s, L=L, h=h: L.ftb_exec_launch(h, C.c_void_p(s.cuda_stream))))
    res = [1e9] * len(graphs)
    for _ in range(int(os.environ.get("ROUNDS", "5"))):
        for i, g in enumerate(graphs):
            res[i] = min(res[i], time_graph(g))
    ref = (A.float() @ (B.float().transpose(-1, -2) if sh.b_layout == "nk" else B.float()))
    err = ((Cm.float() - ref).abs().max() / ref.abs().max()).item()
    print(f"{sh.name:7s} b{sh.batch:4d} M{sh.M:5d} N{sh.N:5d} K{sh.K:5d} tile {tile}: " + " ".join(f"{v:7.2f}" for v in res) + f" us  err {err:.1e}", flush=True)
