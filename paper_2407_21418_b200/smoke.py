"""smoke(): one small Dense plan and one BMM plan through the planner and the
sm_100a executor on cuda:0, checked against the CPU oracle (oracle/execute_np.py)."""

from __future__ import annotations


def run_smoke() -> None:
    import numpy as np
    import torch

    from oracle.execute_np import execute_plan
    from .runtime import Planner
    from .shapeset import ShapeSet
    from .workloads import Shape

    if not torch.cuda.is_available():
        raise RuntimeError("smoke() needs cuda:0")
    shapes = [Shape("dense", "qkv", 1, 160, 2304, 768, "nk"),
              Shape("bmm", "scores", 24, 37, 37, 64, "nk", ("i", "j")),
              Shape("bmm", "context", 24, 37, 64, 37, "kn", ("i", "k"))]
    ss = ShapeSet(shapes, Planner(), device="cuda:0", seed=0)
    ss.launch()
    torch.cuda.synchronize()
    for x, rec in zip(ss.bound, ss.records):
        sh = x.shape
        A = x.A.float().cpu().numpy()
        B = x.B.float().cpu().numpy()
        if sh.b_layout == "nk":
            B = np.swapaxes(B, -1, -2)
        g = rec.program
        space = ["i", "j"] if sh.kind == "dense" else ["b", "i", "j"]
        axes = space + ["k"]
        parts = [({a: int(g.smem[p][d]) for d, a in enumerate(axes)}, int(g.count[p])) for p in range(g.n_parts)]
        ext = {"i": sh.M, "j": sh.N, "b": sh.batch}
        ref, cov = execute_plan(A, B, ext, space, space[g.tau], parts)
        assert (cov == 1).all(), f"{sh.name}: plan does not cover C exactly once"
        got = x.C.float().cpu().numpy()
        err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)
        assert err < 2e-2, f"{sh.name}: rel err {err}"
        print(f"smoke {sh.name} b={sh.batch} M={sh.M} N={sh.N} K={sh.K}: rel err {err:.2e}, "
              f"plan {rec.describe()['parts']}")
    print("smoke ok:", ss.exe.info)
