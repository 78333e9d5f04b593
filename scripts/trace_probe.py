"""Phase trace of the tcgen05 executor on a few shapes (debug aid)."""
import sys, json
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import Shape, c1_shapes

def probe(name, shapes):
    ss = ShapeSet(shapes, Planner(), device="cuda:0")
    ex = ss.exe
    for _ in range(5): ex.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ex.launch(); e1.record(); torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    ex.set_trace(True); ex.launch(); torch.cuda.synchronize(); tr = ex.read_trace().astype(np.int64)
    ex.set_trace(False)
    t0 = tr[tr > 0].min()
    rel = np.where(tr > 0, tr - t0, -1)
    print(f"== {name}: {t_ms*1e3:.1f} us/launch, cfg={ex.config()}, items={ex.info.n_work}, ctas={ex.info.n_ctas}")
    for c in range(min(3, rel.shape[0])):
        for i in range(min(6, rel.shape[1])):
            r = rel[c, i]
            if r[0] < 0: break
            print(f"  cta{c} item{i}: pick {r[0]/1e3:7.2f} k0iss {r[1]/1e3:7.2f} k0land {r[2]/1e3:7.2f} commit {r[3]/1e3:7.2f} epi {r[4]/1e3:7.2f} rel {r[5]/1e3:7.2f} us")
    ok = rel[:, :, 5] >= 0
    print("  mean item (epi release - pick) us:", float(np.mean((rel[:,:,5]-rel[:,:,0])[ok]))/1e3,
          " k0 latency (land - issue) us:", float(np.mean((rel[:,:,2]-rel[:,:,1])[ok]))/1e3,
          " mma->epi us:", float(np.mean((rel[:,:,4]-rel[:,:,3])[ok]))/1e3,
          " epi us:", float(np.mean((rel[:,:,5]-rel[:,:,4])[ok]))/1e3)

probe("qkv M=160", [Shape("dense", "qkv", 1, 160, 2304, 768, "nk")])
probe("ffn1 M=1984", [Shape("dense", "ffn1", 1, 1984, 3072, 768, "nk")])
probe("scores T=62", [Shape("bmm", "scores", 384, 62, 62, 64, "nk", ("i", "j"))])
probe("context T=62", [Shape("bmm", "context", 384, 62, 64, 62, "kn", ("i", "k"))])
probe("C1 step", c1_shapes(24, 0))
