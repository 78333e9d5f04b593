"""Phase trace of ONE shape's launch: where the fixed ~5 us of a small Dense goes.
SHAPE="M N K" (Dense, nk); prints CUDA-event time per launch vs the device
trace span (first producer pick -> last epilogue release) per CTA."""
import os, sys
import os as _os
_os.environ.setdefault("FTB_LIB", "paper_2407_21418_b200/libftb_trace.so")  # phase traces need the trace build (make -C paper_2407_21418_b200/csrc trace)
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.workloads import dense_instance
from paper_2407_21418_b200.calibrate import time_launches
for spec in os.environ.get("SHAPES", "160 768 768;1376 768 768;160 768 3072").split(";"):
    M, N, K = map(int, spec.split())
    A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    rec = Planner().plan([dense_instance(M, N, K)])[0]
    ex = Executable([gemm_desc(A, B, C, "nk")], [rec.program], (A, B, C))
    us = time_launches(lambda s: ex.launch(s), reps=20)
    us1 = time_launches(lambda s: ex.launch(s), reps=1)
    tab = ex.table()
    warm = float(os.environ.get("WARM_S", "0"))
    if warm:
        import time
        t_end = time.time() + warm
        while time.time() < t_end:
            for _ in range(200): ex.launch()
            torch.cuda.synchronize()
        us = time_launches(lambda s: ex.launch(s), reps=20)
        print(f"  after {warm}s warm: {us:.2f} us/launch")
    ex.set_trace(True)
    for _ in range(200 if warm else 1): ex.launch()
    torch.cuda.synchronize()
    tr, kb = ex.read_trace(); tr = tr.astype(np.int64)
    t0 = tr[tr > 0].min()
    rel = np.where(tr > 0, tr - t0, -1) / 1e3
    n = ex.info.n_ctas
    print(f"M{M} N{N} K{K}: {us:.2f} us/launch (graph x20), {us1:.2f} (x1); items {ex.info.n_work}, ctas {n}, cfg {ex.config()['single']}")
    last = rel[:, :, 5].max()
    print(f"  trace span first pick -> last release {last:.2f} us; pick spread {rel[:n,0,0].min():.2f}..{rel[:n,0,0].max():.2f}")
    sp = getattr(ex, "trace_span", None)
    if sp is not None and sp[:n, 1].max() > 0:
        sp = sp[:n].astype(np.int64)
        print(f"  CTA start {((sp[:, 0] - t0) / 1e3).min():.2f}..{((sp[:, 0] - t0) / 1e3).max():.2f} us, "
              f"end p50 {np.median((sp[:, 1] - t0) / 1e3):.2f} max {((sp[:, 1] - t0) / 1e3).max():.2f} us (from first pick)")
    for ev, nm in ((1, "tma0"), (2, "k0land"), (3, "commit"), (4, "epi"), (5, "rel")):
        v = rel[:n, 0, ev]
        print(f"  {nm:7s} min {v.min():.2f} p50 {np.median(v):.2f} max {v.max():.2f}")
    for c in sorted(set([0, n // 2, n - 1])):
        r = rel[c, 0]
        print(f"  cta{c}: pick {r[0]:.2f} tma0 {r[1]:.2f} k0land {r[2]:.2f} commit {r[3]:.2f} epi {r[4]:.2f} rel {r[5]:.2f}")
    kbr = np.where(kb > 0, kb.astype(np.int64) - t0, -1) / 1e3
    for c in sorted(set([0, n - 1])):
        print(f"  cta{c} kb issue:", " ".join(f"{v:.2f}" for v in kbr[c, :16, 0]))
        print(f"  cta{c} kb mma  :", " ".join(f"{v:.2f}" for v in kbr[c, :16, 1]))
    if os.environ.get("EPI"):
        ep = kb[:n, 40:46, :].reshape(n, 12).astype(np.int64)
        d = np.diff(ep, axis=1)
        print("  epi clk deltas (ld->waitread, ->staged, ->fenced, ->store0, ->store1+commit, ->ld1, ...) median over CTAs:",
              np.median(d, axis=0).astype(int).tolist())
        print("  rel - epi per CTA p50:", f"{np.median(rel[:n,0,5]-rel[:n,0,4]):.2f}")
    ex.close()
