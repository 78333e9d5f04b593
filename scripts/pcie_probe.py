import torch
n = 822091776 // 2
h_in = torch.empty(n, dtype=torch.bfloat16).pin_memory(); h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d_in = torch.empty(n, dtype=torch.bfloat16, device="cuda"); d_out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d(): d_in.copy_(h_in, non_blocking=True)
def d2h(): h_out.copy_(d_out, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
b = n * 2
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.2f} ms  {b / ms / 1e6:.1f} GB/s per direction")


# chunked: each direction split into C pieces on C streams (several copy engines)
def chunked(C):
    hs = [torch.cuda.Stream() for _ in range(C)]
    ds = [torch.cuda.Stream() for _ in range(C)]
    step = (n + C - 1) // C

    def fn():
        cur = torch.cuda.current_stream()
        for s in hs + ds:
            s.wait_stream(cur)
        for c in range(C):
            lo, hi = c * step, min(n, (c + 1) * step)
            with torch.cuda.stream(hs[c]):
                d_in[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
            with torch.cuda.stream(ds[c]):
                h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
        for s in hs + ds:
            cur.wait_stream(s)
    return fn


for C in (2, 4, 8):
    ms = t(chunked(C))
    print(f"both, {C} chunks per direction: {ms:.2f} ms  {b / ms / 1e6:.1f} GB/s per direction")
