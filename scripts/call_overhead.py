"""Host cost of one Planner.dense / .bmm call on a warm cache (cProfile + wall)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2407_21418_b200.runtime import Planner  # noqa: E402

pl = Planner()
A = torch.randn(32 * 40, 768, device="cuda").bfloat16()
W = torch.randn(2304, 768, device="cuda").bfloat16()
b = torch.randn(2304, device="cuda").bfloat16()
out = torch.empty(32 * 40, 2304, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    pl.dense(A, W, b_layout="nk", bias=b, out=out)
    pl.dense(A, W, b_layout="nk", bias=b)
torch.cuda.synchronize()
for label, kw in (("out=given", {"out": out}), ("out=None", {})):
    t0 = time.perf_counter()
    for _ in range(200):
        pl.dense(A, W, b_layout="nk", bias=b, **kw)
    torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us per call")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    pl.dense(A, W, b_layout="nk", bias=b, out=out)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
