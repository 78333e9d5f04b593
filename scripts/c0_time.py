"""C0 (fp32 FFMA validation mode, N = K = 768) per-shape timing: L2-cold PDL
chain (as bench.py) of the FFMA executor vs cuBLAS fp32 (TF32 off) on the
same shapes; roofline = max(F / 74.45 TF/s FFMA peak, bytes / 8 TB/s).
  MS="1 16 64 128 256 509 512" python scripts/c0_time.py"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2407_21418_b200.execute import Executable, gemm_desc  # noqa: E402
from paper_2407_21418_b200.mktune.hardware import b200_ffma  # noqa: E402
from paper_2407_21418_b200.runtime import Planner, dense_instance  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
P = 148 * 128 * 2 * 1.965e9
pl = Planner(hw=b200_ffma())


def chain(launches, n):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for f in launches:
            f(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for f in launches:
            f(s)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    return sorted(ts)[2]


for M in map(int, os.environ.get("MS", "1 16 64 128 256 509 512").split()):
    N = K = 768
    byts = 4 * (M * K + K * N + M * N)
    n = max(20, min(512, -(-252_000_000 // byts)))
    bufs = [((torch.rand(M, K, device="cuda") - .5), (torch.rand(K, N, device="cuda") - .5),
             torch.empty(M, N, device="cuda")) for _ in range(n)]
    rec = pl.plan([dense_instance(M, N, K, elem_bytes=4, m_max=512)])[0]
    exes = [Executable([gemm_desc(A, B, C, "kn")], [rec.program]) for A, B, C in bufs]
    t_ours = chain([lambda s, e=e: e.launch(s) for e in exes], n)
    t_cub = chain([lambda s, A=A, B=B, C=C: torch.matmul(A, B, out=C) for A, B, C in bufs], n)
    roof = max(2 * M * N * K / P, byts / 8e12) * 1e6
    print(f"C0 M={M:4d}: ours {t_ours:7.2f} us ({2 * M * N * K / t_ours / 1e6:6.2f} TF/s, roofline frac {roof / t_ours:.3f}, "
          f"items {exes[0].info.n_work}, ctas {exes[0].info.n_ctas})  cuBLAS fp32 {t_cub:7.2f} us (frac {roof / t_cub:.3f})",
          flush=True)
