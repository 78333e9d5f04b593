"""8192^3 (and 4096^3) bf16 GEMM: this executor vs torch.matmul (cuBLAS),
sustained (2 s of back-to-back launches each), with nvidia-smi SM clock
samples during each run: separates per-clock efficiency from power state."""
import subprocess, sys, threading, time
sys.path.insert(0, ".")
import torch
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner, dense_instance


def sample_clocks(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        try:
            out.append(int(r.stdout.strip().splitlines()[0]))
        except Exception:
            pass
        time.sleep(0.1)


def run(name, fn, flops, secs=2.0):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    clk, stop = [], threading.Event()
    th = threading.Thread(target=sample_clocks, args=(stop, clk)); th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0; t_end = time.time() + secs
    e0.record()
    while time.time() < t_end:
        for _ in range(10): fn()
        n += 10
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    us = e0.elapsed_time(e1) * 1e3 / n
    mhz = sorted(clk)[len(clk) // 2] if clk else 0
    tf = flops / (us * 1e-6) / 1e12
    print(f"{name}: {us:.1f} us  {tf:.0f} TF/s  SM {mhz} MHz  -> {tf * 1e12 / (148 * mhz * 1e6):.0f} flop/clk/SM", flush=True)


import os
for spec in os.environ.get("SHAPES", "8192 8192 8192;4096 4096 4096").split(";"):
    M, N, K = map(int, spec.split())
    A = torch.randn(M, K, device="cuda").bfloat16(); B = torch.randn(N, K, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ex = Executable([gemm_desc(A, B, C, "nk")], [Planner().plan([dense_instance(M, N, K)])[0].program], (A, B, C))
    fl = 2 * M * N * K
    run(f"ours   {M}x{N}x{K}", lambda: ex.launch(), fl)
    run(f"cuBLAS {M}x{N}x{K}", lambda: torch.matmul(A, B.t(), out=C), fl)
    run(f"ours   {M}x{N}x{K}", lambda: ex.launch(), fl)
    ex.close()
