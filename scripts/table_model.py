"""Offline cost model of a lowered C1 table (CPU only): per-item MMA clocks
with the measured B200 issue floor (~100 clk per M=128 K=16 tcgen05.mma,
N/2 clk above N=200) and TMA ingest (~110 B/clk/SM)."""
import sys, collections
sys.path.insert(0, ".")
import numpy as np
from paper_2407_21418_b200.execute import lower_table, gemm_desc
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.workloads import c1_shapes
from paper_2407_21418_b200 import _lib

def model(shapes, planner, label):
    recs = planner.plan([s.instance() for s in shapes])
    tot = collections.Counter(); nitems = collections.Counter(); ideal = collections.Counter()
    for s, r in zip(shapes, recs):
        items, info = lower_table_for(s, r.program)
        for (p, b, l0, c0, ll, cl, n, _) in items:
            kb = -(-s.K // 64)
            t_mma = 4 * max(100, n / 2)
            t_tma = (128 + n) * 128 / 110
            tot[s.kind] += kb * max(t_mma, t_tma)
            nitems[s.kind] += 1
        ideal[s.kind] += s.flops / 8192 / 2  # clk at 8192 flop/clk/SM... per SM-sum: flops/(8192)
    for k in tot:
        print(f"{label:10s} {k:6s} items {nitems[k]:6d}  model SM-clk {tot[k]/1e6:8.2f}M  -> {tot[k]/148/1.9e9*1e3:7.3f} ms at 1.9GHz/148 SMs;  ideal {ideal[k]*2/148/1.9e9*1e3:7.3f} ms")

def lower_table_for(s, prog):
    import ctypes as C
    d = _lib.GemmDesc()
    d.op = 0 if s.kind == "dense" else 1
    d.batch = s.batch; d.M = s.M; d.N = s.N; d.K = s.K
    d.A = 16; d.B = 16; d.C = 16
    d.lda = (s.K + 7) // 8 * 8; d.ldb = s.K if s.b_layout == "nk" else (s.N + 7) // 8 * 8; d.ldc = (s.N + 7) // 8 * 8
    d.a_batch_stride = s.M * d.lda; d.b_batch_stride = (s.N if s.b_layout == "nk" else s.K) * d.ldb; d.c_batch_stride = s.M * d.ldc
    d.in_dtype = 0; d.out_dtype = 0; d.b_layout = 1 if s.b_layout == "nk" else 0; d.orientation = -1
    items, info = lower_table([d], [prog])
    return items.tolist(), info

if __name__ == "__main__":
    shapes = c1_shapes(24, 0)
    model(shapes, Planner(), "default")
