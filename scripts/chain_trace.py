"""Where the per-launch floor of a small shape goes: a PDL chain of launches
of ONE shape on distinct buffers (as bench.py's per-shape timing runs it),
each launch traced (trace build: make -C paper_2407_21418_b200/csrc trace).

For each launch k prints, in us relative to launch 0's first CTA start:
CTA start (min..max), producer pick, first TMA issue, K block 0 landed, MMA
commit, epilogue start, epilogue release, CTA end (p50 / max) and the gap
between launch k's last CTA end and launch k+1's first TMA issue.

  SHAPE="bmm 384 5 5 64 nk" | "dense 160 768 768" python scripts/chain_trace.py
"""
import os
import sys

os.environ.setdefault("FTB_LIB", "paper_2407_21418_b200/libftb_trace.so")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_21418_b200.execute import Executable, gemm_desc  # noqa: E402
from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance  # noqa: E402

NL = int(os.environ.get("NL", "6"))
for spec in os.environ.get("SHAPES", "bmm 384 5 5 64 nk;bmm 384 100 100 64 nk;dense 608 768 768;dense 160 768 3072").split(";"):
    f = spec.split()
    if f[0] == "bmm":
        b, M, N, K, lay = int(f[1]), int(f[2]), int(f[3]), int(f[4]), f[5]
        inst = bmm_instance(b, M, N, K, ("i", "j") if lay == "nk" else ("i", "k"))
        mk = lambda: ((torch.rand(b, M, K, device="cuda") * 2 - 1).bfloat16(),  # noqa: E731
                      (torch.rand(b, N, K, device="cuda") * 2 - 1).bfloat16() if lay == "nk"
                      else (torch.rand(b, K, N, device="cuda") * 2 - 1).bfloat16(),
                      torch.empty(b, M, N, device="cuda", dtype=torch.bfloat16))
    else:
        M, N, K, lay = int(f[1]), int(f[2]), int(f[3]), "nk"
        inst = dense_instance(M, N, K)
        mk = lambda: ((torch.rand(M, K, device="cuda") * 2 - 1).bfloat16(),  # noqa: E731
                      (torch.rand(N, K, device="cuda") * 2 - 1).bfloat16(),
                      torch.empty(M, N, device="cuda", dtype=torch.bfloat16))
    rec = Planner().plan([inst])[0]
    bufs = [mk() for _ in range(NL)]
    exes = [Executable([gemm_desc(A, B, C, lay)], [rec.program], (A, B, C)) for A, B, C in bufs]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for e in exes:
            e.launch(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for e in exes:
            e.launch(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us_plain = e0.elapsed_time(e1) * 1e3 / NL
    for e in exes:
        e.set_trace(True)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        for e in exes:
            e.launch(s)
    for _ in range(2):
        g2.replay()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        e0.record(s)
        g2.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us_trace = e0.elapsed_time(e1) * 1e3 / NL
    n = exes[0].info.n_ctas
    print(f"{spec}: {us_plain:.2f} us/launch (release build path {os.environ['FTB_LIB']}), traced {us_trace:.2f}; "
          f"items {exes[0].info.n_work} ctas {n} cfg {exes[0].config()['single']}")
    traces = []
    for e in exes:
        tr, kb_ = e.read_trace()
        traces.append((tr.astype(np.int64)[:n], e.trace_span.astype(np.int64)[:n], kb_[:n]))
    t0 = min(sp[:, 0][sp[:, 0] > 0].min() for _, sp, _ in traces)
    prev_end = None
    for k, (tr, sp, kb) in enumerate(traces):
        r = np.where(tr > 0, tr - t0, -1) / 1e3
        st = (sp[:, 0] - t0) / 1e3
        en = (sp[:, 1] - t0) / 1e3
        first_tma = r[:, 0, 1][r[:, 0, 1] >= 0].min()
        gap = "" if prev_end is None else f" gap(prev end -> tma0) {first_tma - prev_end:+.2f}"
        print(f"  L{k}: start {st.min():6.2f}..{st.max():6.2f} pick {np.median(r[:, 0, 0]):6.2f} "
              f"tma0 {first_tma:6.2f}/{np.median(r[:, 0, 1]):6.2f} k0land {np.median(r[:, 0, 2]):6.2f} "
              f"commit {np.median(r[:, 0, 3]):6.2f} epi {np.median(r[:, 0, 4]):6.2f} rel {np.median(r[:, 0, 5]):6.2f} "
              f"end p50 {np.median(en):6.2f} max {en.max():6.2f}{gap}")
        prev_end = en.max()
        if os.environ.get("CL"):  # clock64 stamps (same SM): sync1, reduce, sync2 durations in clk
            c = kb[:, 60:62, :].reshape(len(kb), 4).astype(np.int64)
            d = np.diff(c, axis=1)
            print(f"     cluster clk: sync1 p50 {np.median(d[:, 0]):.0f} max {d[:, 0].max():.0f} | reduce p50 "
                  f"{np.median(d[:, 1]):.0f} max {d[:, 1].max():.0f} | sync2 p50 {np.median(d[:, 2]):.0f} max {d[:, 2].max():.0f}")
            x = kb[:, 62:64, :].reshape(len(kb), 4).astype(np.int64)  # 124 summed, 125 stored, 126 entry
            red = (x[:, 2] > 0) & (x[:, 0] > 0)
            if red.any():
                r0 = c[red, 1]
                print(f"     reducing CTAs: entry-after-sync1 {np.median(x[red, 2] - r0):.0f} | loads+sum {np.median(x[red, 0] - x[red, 2]):.0f}"
                      f" | stage+store issue {np.median(x[red, 1] - x[red, 0]):.0f} | rest {np.median(c[red, 2] - x[red, 1]):.0f} clk")
        if os.environ.get("KB"):
            kbr = np.where(kb > 0, kb.astype(np.int64) - t0, -1) / 1e3
            print("     kb issue-stamp:", " ".join(f"{v:.2f}" for v in kbr[0, :8, 0]), "| mma saw:",
                  " ".join(f"{v:.2f}" for v in kbr[0, :8, 1]))
