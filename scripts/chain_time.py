"""Per-launch time of a PDL chain of ONE shape on NL distinct buffer sets
(CUDA graph, L2-cold when NL * bytes > L2), release library.

  SHAPES="dense 608 768 768;bmm 384 5 5 64 nk" NL=64 python scripts/chain_time.py
Env knobs of the executor (FTB_TMA_STORE, FTB_EPI8, FTB_SPLITK, ...) are read
at table creation, so set them on the command line."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2407_21418_b200.execute import Executable, gemm_desc  # noqa: E402
from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance  # noqa: E402

NL = int(os.environ.get("NL", "20"))
for spec in os.environ.get("SHAPES", "dense 128 256 64;dense 608 768 768;bmm 384 5 5 64 nk").split(";"):
    f = spec.split()
    if f[0] == "bmm":
        b, M, N, K, lay = int(f[1]), int(f[2]), int(f[3]), int(f[4]), f[5]
        inst = bmm_instance(b, M, N, K, ("i", "j") if lay == "nk" else ("i", "k"))
        Np = (N + 7) // 8 * 8

        def mk():
            Kp = (K + 7) // 8 * 8
            A = (torch.rand(b, M, Kp, device="cuda") * 2 - 1).bfloat16()[:, :, :K]
            B = ((torch.rand(b, N, K, device="cuda") if lay == "nk" else torch.rand(b, K, N, device="cuda")) * 2 - 1).bfloat16()
            C = torch.empty(b, M, Np, device="cuda", dtype=torch.bfloat16)[:, :, :N]
            return A, B, C
    else:
        M, N, K, lay = int(f[1]), int(f[2]), int(f[3]), "nk"
        inst = dense_instance(M, N, K)

        def mk():
            return ((torch.rand(M, K, device="cuda") * 2 - 1).bfloat16(), (torch.rand(N, K, device="cuda") * 2 - 1).bfloat16(),
                    torch.empty(M, N, device="cuda", dtype=torch.bfloat16))
    rec = Planner().plan([inst])[0]
    nl = NL
    if os.environ.get("COLD", "1") == "1":  # as bench.py: copies totalling >= 252 MB (2x L2)
        a, bb, c = mk()
        byts = sum(t.numel() * t.element_size() for t in (a, bb, c))
        nl = max(NL, min(1024, -(-252_000_000 // byts)))
    bufs = [mk() for _ in range(nl)]
    exes = [Executable([gemm_desc(A, B, C, lay)], [rec.program]) for A, B, C in bufs]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for e in exes:
            e.launch(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for e in exes:
            e.launch(s)
    ts = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / nl)
    ts.sort()
    env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FTB_"))
    print(f"{spec:28s} {ts[len(ts) // 2]:6.2f} us/launch  chain {nl:4d}  items {exes[0].info.n_work:4d} ctas {exes[0].info.n_ctas:3d} kernel-items {exes[0].config()['n_singles']:4d} split {exes[0].config()['cluster_split']}{'w' if exes[0].config()['workspace_split'] else 'c'} "
          f"cfg {exes[0].config()['single']}  [{env}]", flush=True)
