import os, sys
import os as _os
_os.environ.setdefault("FTB_LIB", "paper_2407_21418_b200/libftb_trace.so")  # phase traces need the trace build (make -C paper_2407_21418_b200/csrc trace)
os.environ.setdefault("FTB_PAIR", "0")
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.workloads import Shape

def run(name, M, N, K, prog):
    A = (torch.rand(M, K, device="cuda") - 0.5).bfloat16(); B = (torch.rand(N, K, device="cuda") - 0.5).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ex = Executable([gemm_desc(A, B, C, "nk")], [prog], (A, B, C))
    for _ in range(5): ex.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ex.launch(); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e3
    ex.set_trace(True)
    ex.launch(); torch.cuda.synchronize()
    tr, kb = ex.read_trace(); tr = tr.astype(np.int64); kb = kb.astype(np.int64)
    t0 = min(tr[tr > 0].min(), kb[kb > 0].min())
    rel = np.where(tr > 0, tr - t0, -1) / 1e3
    kr = np.where(kb > 0, kb - t0, -1) / 1e3
    print(f"== {name} M{M} N{N} K{K}: {t:.1f} us (events), items {ex.info.n_work} ctas {ex.info.n_ctas} cfg {ex.config()}")
    for c in (0, 1, min(100, rel.shape[0]-1)):
        for i in range(4):
            r = rel[c, i]
            if r[0] < 0: break
            print(f"  cta{c} it{i}: pick {r[0]:6.2f} k0iss {r[1]:6.2f} k0land {r[2]:6.2f} commit {r[3]:6.2f} epi {r[4]:6.2f} rel {r[5]:6.2f}")
        print(f"  cta{c} kb issue:", " ".join(f"{v:5.2f}" for v in kr[c, :48, 0]))
        print(f"  cta{c} kb land :", " ".join(f"{v:5.2f}" for v in kr[c, :48, 1]))
    print(f"  last release {rel[:, :, 5].max():.2f} us")
    ex.set_trace(False)

pl = Planner()
if os.environ.get("ONE"):
    M, N, K = (int(x) for x in os.environ["ONE"].split(","))
    rec = pl.plan([Shape("dense", "one", 1, M, N, K, "nk").instance()])[0]
    run("plan", M, N, K, rec.program)
    sys.exit(0)
if os.environ.get("BIGONLY"):
    run("ffn1 256x256", 4096, 3072, 768, program_struct(2, 0, [((1, 1), (256, 256, 64), 16)]))
    run("4096 256x256", 4096, 4096, 4096, program_struct(2, 0, [((1, 1), (256, 256, 64), 16)]))
    sys.exit(0)
for (name, M, N, K) in [("ffn2", 768, 768, 3072), ("ffn2", 160, 768, 3072), ("ffn1", 4096, 3072, 768)]:
    rec = pl.plan([Shape("dense", name, 1, M, N, K, "nk").instance()])[0]
    run(name + " plan", M, N, K, rec.program)
run("ffn1 128x256", 4096, 3072, 768, program_struct(2, 0, [((1, 1), (128, 256, 64), 32)]))
run("big 128x256", 8192, 8192, 8192, program_struct(2, 0, [((1, 1), (128, 256, 64), 64)]))
