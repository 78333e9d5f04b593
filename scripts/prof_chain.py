"""clock64 role profile (FTB_PROD_PROFILE build, libftb_prof.so) of the LAST
launch of an L2-cold chain of one shape: per CTA the producer's wait-for-slot
/ issue cycles, the MMA warp's wait-for-TMEM / wait-for-data / issue cycles
and the epilogue's wait, averaged over CTAs (cycles at the SM clock).
  SHAPES="dense 16 4096 4096" python scripts/prof_chain.py"""
import os
import sys

os.environ.setdefault("FTB_LIB", "paper_2407_21418_b200/libftb_prof.so")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_21418_b200.execute import Executable, gemm_desc  # noqa: E402
from paper_2407_21418_b200.runtime import Planner, dense_instance, bmm_instance  # noqa: E402

for spec in os.environ.get("SHAPES", "dense 16 4096 4096").split(";"):
    f = spec.split()
    if f[0] == "bmm":
        b, M, N, K, lay = int(f[1]), int(f[2]), int(f[3]), int(f[4]), f[5]
        inst = bmm_instance(b, M, N, K, ("i", "j") if lay == "nk" else ("i", "k"))
        Np = (N + 7) // 8 * 8
        mk = lambda: ((torch.rand(b, M, K, device="cuda") - .5).bfloat16(),  # noqa: E731
                      ((torch.rand(b, N, K, device="cuda") if lay == "nk" else torch.rand(b, K, N, device="cuda")) - .5).bfloat16(),
                      torch.empty(b, M, Np, device="cuda", dtype=torch.bfloat16)[:, :, :N])
    else:
        M, N, K, lay = int(f[1]), int(f[2]), int(f[3]), "nk"
        inst = dense_instance(M, N, K)
        mk = lambda: ((torch.rand(M, K, device="cuda") - .5).bfloat16(), (torch.rand(N, K, device="cuda") - .5).bfloat16(),  # noqa: E731
                      torch.empty(M, N, device="cuda", dtype=torch.bfloat16))
    rec = Planner().plan([inst])[0]
    a, bb, c = mk()
    nl = max(8, min(256, -(-252_000_000 // sum(t.numel() * 2 for t in (a, bb, c)))))
    exes = [Executable([gemm_desc(*mk(), lay)], [rec.program]) for _ in range(nl)]
    for e in exes:
        e.set_trace(True)
    s = torch.cuda.Stream()
    for rep in range(3):
        with torch.cuda.stream(s):
            for e in exes:
                e.launch(s)
        torch.cuda.synchronize()
    tr, _ = exes[-1].read_trace()
    n = exes[-1].info.n_ctas
    raw = tr.reshape(tr.shape[0], -1)[:n, :12].astype(np.float64)
    p_wait, p_issue, p_item, nkb, nitems, p_total, m_te, m_full, m_issue, m_total, e_wait, e_total = raw.T
    print(f"{spec}: ctas {n} items/CTA {nitems.mean():.1f} kb/CTA {nkb.mean():.1f} cfg {exes[-1].config()['single']}")
    print(f"  producer: wait-slot {p_wait.mean():.0f} issue {p_issue.mean():.0f} total {p_total.mean():.0f} clk "
          f"(per kb: wait {np.mean(p_wait / np.maximum(nkb, 1)):.0f}, issue {np.mean(p_issue / np.maximum(nkb, 1)):.0f})")
    print(f"  mma     : wait-tmem {m_te.mean():.0f} wait-data {m_full.mean():.0f} issue {m_issue.mean():.0f} total {m_total.mean():.0f}")
    print(f"  epilogue: wait-acc {e_wait.mean():.0f} total {e_total.mean():.0f}  (max total {e_total.max():.0f})")
