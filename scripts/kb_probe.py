"""Per-K-block producer/MMA timing for a big GEMM (single-CTA kernel)."""
import os, sys
os.environ["FTB_PAIR"] = "0"
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct
for (M, N, K, ti, tj) in [(8192, 8192, 8192, 128, 256), (2048, 2304, 768, 128, 128)]:
    A = (torch.rand(M, K, device="cuda") - 0.5).bfloat16(); B = (torch.rand(N, K, device="cuda") - 0.5).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ex = Executable([gemm_desc(A, B, C, "nk", orientation=0)], [program_struct(2, 0, [((1, 1), (ti, tj, 64), M // ti)])], (A, B, C))
    for _ in range(3): ex.launch()
    torch.cuda.synchronize()
    ex.set_trace(True); ex.launch(); torch.cuda.synchronize()
    items, kb = ex.read_trace()
    kb = kb.astype(np.int64)
    t0 = kb[kb > 0].min()
    print(f"== M{M} N{N} K{K} {ti}x{tj} cfg {ex.config()['single']}")
    for c in (0, 1, 77):
        iss = (kb[c, :, 0] - t0) / 1e3; see = (kb[c, :, 1] - t0) / 1e3
        print(f" cta{c} issue:", " ".join(f"{v:6.2f}" for v in iss[:24]))
        print(f" cta{c}  seen:", " ".join(f"{v:6.2f}" for v in see[:24]))
        d = np.diff(see[8:60]); print(f"   steady MMA-side gap mean {d.mean()*1e3:.0f} ns; issue->seen latency mean {(see-iss)[8:60].mean()*1e3:.0f} ns")
