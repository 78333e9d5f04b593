S="dense 16 4096 4096;dense 64 4096 4096;dense 256 4096 4096"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2v.txt 2>&1
SHAPES="$S" FTB_SPLIT_CLUSTER=0 python scripts/chain_time.py >> gpurun_out/r2v.txt 2>&1
SHAPES="$S" FTB_SPLITK=0 python scripts/chain_time.py >> gpurun_out/r2v.txt 2>&1
CL=1 SHAPES="dense 16 4096 4096" NL=4 python scripts/chain_trace.py >> gpurun_out/r2v.txt 2>&1
python scripts/cublas_step.py > /dev/null 2>&1 || true
python - >> gpurun_out/r2v.txt 2>&1 <<'PY'
import torch
for M in (16, 64, 256):
    n = max(20, -(-252_000_000 // (4096*4096*2 + M*4096*4)))
    As=[torch.randn(M,4096,device='cuda').bfloat16() for _ in range(n)]; Ws=[torch.randn(4096,4096,device='cuda').bfloat16() for _ in range(n)]
    s=torch.cuda.Stream()
    with torch.cuda.stream(s):
        for a,w in zip(As,Ws): torch.matmul(a,w.t())
    torch.cuda.synchronize()
    g=torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for a,w in zip(As,Ws): torch.matmul(a,w.t())
    g.replay(); torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(f"cublas dense {M} 4096 4096 L2-cold chain {n}: {e0.elapsed_time(e1)*1e3/n:.2f} us")
PY
cat gpurun_out/r2v.txt | cut -c 1-220
