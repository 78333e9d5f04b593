"""Randomised parity sweep on B200 (seeded). Each case draws a few dozen
problems: Dense or BatchMatmul, ragged extents (M, N, K from 1 up),
both B layouts, bf16 or fp32 outputs, fused bias (bf16/fp32) and GELU on
Dense, operands and outputs with padded row strides. Every problem is
planned by the B200 planner (fallback ladder included) and executed
(a) alone, one launch each, and (b) all together in ONE grouped table.
Both must match a float64 reference of the same op per element
(tests/_numerics.py), and neither may write outside its output view: the padding
columns of every output (and the gap rows between batch entries) stay NaN."""

import math
import random

import pytest
import torch
import torch.nn.functional as F

from _numerics import check
from paper_2407_21418_b200.execute import Executable, gemm_desc
from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance

pytestmark = pytest.mark.gpu



def _padded(shape, dtype, dev, g, fill=None):
    """A view of `shape` whose rows are padded to a multiple of 8 elements
    (+ 8 more), so its last dim is contiguous and strides are TMA-legal."""
    *lead, cols = shape
    ld = (cols + 7) // 8 * 8 + 8
    if fill is None:
        base = (torch.rand(*lead, ld, generator=g) * 2 - 1).to(dtype).to(dev)
    else:
        base = torch.full((*lead, ld), fill, dtype=dtype, device=dev)
    return base, base[..., :cols]


def _draw(rng, g, dev):
    dense = rng.random() < 0.55
    b_layout = rng.choice(["kn", "nk"])
    out_dtype = torch.float32 if rng.random() < 0.2 else torch.bfloat16
    if dense:
        M = int(math.exp(rng.uniform(0.0, math.log(3000.0))))
        N = rng.choice([1, 24, 64, 96, 200, 256, 520, 768, 1000, 2304])
        K = rng.choice([5, 40, 64, 100, 256, 768, 1500])
        A_base, A = _padded((M, K), torch.bfloat16, dev, g)
        B_base, B = _padded((K, N) if b_layout == "kn" else (N, K), torch.bfloat16, dev, g)
        C_base, C = _padded((M, N), out_dtype, dev, g, fill=float("nan"))
        bias = act = None
        if rng.random() < 0.35:
            bias = ((torch.rand(N, generator=g) * 2 - 1) * 0.5).to(rng.choice([torch.bfloat16, torch.float32])).to(dev)
            act = "gelu" if rng.random() < 0.5 else None
        inst = dense_instance(M, N, K)
        Bkn = B.double() if b_layout == "kn" else B.double().t()
        ref = A.double() @ Bkn
        if bias is not None:
            ref = ref + bias.double()
        if act == "gelu":
            ref = F.gelu(ref)
        return dict(inst=inst, A=A, B=B, C=C, C_base=C_base, b_layout=b_layout, bias=bias, act=act, ref=ref, K=K,
                    keep=(A_base, B_base, C_base), name=f"dense M{M} N{N} K{K} {b_layout} {out_dtype} bias={bias is not None} {act}")
    b = rng.choice([1, 3, 12, 40])
    kind = rng.choice(["scores", "context", "free"])
    T = rng.randint(1, 300)
    if kind == "scores":
        M, N, K, dyn = T, T, 64, ("i", "j")
    elif kind == "context":
        M, N, K, dyn = T, 64, T, ("i", "k")
    else:
        M, N, K, dyn = rng.randint(1, 300), rng.randint(1, 300), rng.randint(1, 300), ("i", "j")
    A_base, A = _padded((b, M, K), torch.bfloat16, dev, g)
    B_base, B = _padded((b, K, N) if b_layout == "kn" else (b, N, K), torch.bfloat16, dev, g)
    C_base, C = _padded((b, M, N), out_dtype, dev, g, fill=float("nan"))
    Bkn = B.double() if b_layout == "kn" else B.double().transpose(1, 2)
    return dict(inst=bmm_instance(b, M, N, K, dyn), A=A, B=B, C=C, C_base=C_base, b_layout=b_layout, bias=None,
                act=None, ref=A.double() @ Bkn, K=K, keep=(A_base, B_base, C_base),
                name=f"bmm {kind} b{b} M{M} N{N} K{K} {b_layout} {out_dtype}")


def _check(p, tag):
    C = p["C"]
    assert not torch.isnan(C.float()).any(), f"{tag}: unwritten outputs in {p['name']}"
    # per element: 8e-3 relative + a sqrt(K)-scaled accumulation term
    # (tests/_numerics.py); GELU's slope (<= 1.13) scales the latter
    ok, worst, idx = check(C, p["ref"], p["K"], scale=1.2 if p.get("act") else 1.0)
    assert ok, f"{tag}: worst err/tol {worst:.3g} at {idx} in {p['name']}"
    pad = p["C_base"][..., C.shape[-1]:]
    assert torch.isnan(pad.float()).all(), f"{tag}: writes past the output view in {p['name']}"


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_random_problems_alone_and_grouped(cuda, seed):
    rng = random.Random(seed)
    g = torch.Generator(device="cpu").manual_seed(seed)
    probs = [_draw(rng, g, cuda) for _ in range(32)]
    planner = Planner()
    recs = planner.plan([p["inst"] for p in probs])
    # (a) one launch per problem
    for p, r in zip(probs, recs):
        ex = Executable([gemm_desc(p["A"], p["B"], p["C"], p["b_layout"], bias=p["bias"], activation=p["act"])],
                        [r.program], p["keep"])
        ex.launch()
        torch.cuda.synchronize()
        _check(p, "alone")
        ex.close()
    # (b) the same problems as one grouped table
    for p in probs:
        p["C_base"].fill_(float("nan"))
    descs = [gemm_desc(p["A"], p["B"], p["C"], p["b_layout"], bias=p["bias"], activation=p["act"]) for p in probs]
    ex = Executable(descs, [r.program for r in recs], [t for p in probs for t in p["keep"]])
    ex.launch()
    torch.cuda.synchronize()
    for p in probs:
        _check(p, "grouped")
    ex.close()


@pytest.mark.parametrize("mode", ["FTB_TMA_STORE=0", "FTB_SPLITK=0", "FTB_COLSPLIT=0", "FTB_PAIR=1", "FTB_NO_PACK=1"])
@pytest.mark.parametrize("orientation", [0, 1])
def test_random_problems_forced_orientation_and_modes(cuda, monkeypatch, mode, orientation):
    """The same sweep with the orientation forced (0 normal, 1 swap-AB) and
    one executor switch flipped, one grouped table per case."""
    k, v = mode.split("=")
    monkeypatch.setenv(k, v)
    seed = 100 + 10 * orientation + len(mode)
    rng = random.Random(seed)
    g = torch.Generator(device="cpu").manual_seed(seed)
    probs = [_draw(rng, g, cuda) for _ in range(24)]
    recs = Planner().plan([p["inst"] for p in probs])
    descs = [gemm_desc(p["A"], p["B"], p["C"], p["b_layout"], orientation=orientation, bias=p["bias"],
                       activation=p["act"]) for p in probs]
    ex = Executable(descs, [r.program for r in recs], [t for p in probs for t in p["keep"]])
    ex.launch()
    torch.cuda.synchronize()
    for p in probs:
        _check(p, f"{mode} orientation={orientation}")
    ex.close()


@pytest.mark.parametrize("seed", [7, 8])
def test_random_fp32_ffma_problems(cuda, seed):
    """fp32 validation mode (config C0 family): random Dense extents and
    layouts on the FFMA kernel, per element 1e-5 relative against float64."""
    from paper_2407_21418_b200.runtime import dense_instance

    rng = random.Random(seed)
    g = torch.Generator(device="cpu").manual_seed(seed)
    planner = Planner(hw=__import__("paper_2407_21418_b200.mktune.hardware", fromlist=["b200_ffma"]).b200_ffma())
    for _ in range(12):
        M, N, K = rng.randint(1, 600), rng.choice([1, 33, 64, 100, 768]), rng.choice([1, 7, 64, 300, 768])
        b_layout = rng.choice(["kn", "nk"])
        A_base, A = _padded((M, K), torch.float32, cuda, g)
        B_base, B = _padded((K, N) if b_layout == "kn" else (N, K), torch.float32, cuda, g)
        C_base, C = _padded((M, N), torch.float32, cuda, g, fill=float("nan"))
        rec = planner.plan([dense_instance(M, N, K, elem_bytes=4, m_max=512)])[0]
        ex = Executable([gemm_desc(A, B, C, b_layout)], [rec.program], (A_base, B_base, C_base))
        ex.launch()
        torch.cuda.synchronize()
        ref = A.double() @ (B.double() if b_layout == "kn" else B.double().t())
        ok, worst, idx = check(C, ref, K, ffma=True)
        assert ok, (M, N, K, b_layout, worst, idx)
        assert torch.isnan(C_base[:, N:]).all()
        ex.close()


def _draw_large(rng, g, dev):
    """Bigger extents: Dense M up to 8192 with K up to 4096 (split-K for the
    small-table cases, fused bias/GELU, fp32 outputs), BMM batch up to 1024
    with T up to 512 (C2's range), both layouts."""
    if rng.random() < 0.5:
        M = int(math.exp(rng.uniform(0.0, math.log(8192.0))))
        N = rng.choice([128, 768, 1000, 2304, 3072, 4096])
        K = rng.choice([768, 1000, 3072, 4096])
        b_layout = rng.choice(["kn", "nk"])
        out_dtype = torch.float32 if rng.random() < 0.2 else torch.bfloat16
        A_base, A = _padded((M, K), torch.bfloat16, dev, g)
        B_base, B = _padded((K, N) if b_layout == "kn" else (N, K), torch.bfloat16, dev, g)
        C_base, C = _padded((M, N), out_dtype, dev, g, fill=float("nan"))
        bias = act = None
        if rng.random() < 0.4:
            bias = ((torch.rand(N, generator=g) * 2 - 1) * 0.5).to(torch.bfloat16).to(dev)
            act = "gelu" if rng.random() < 0.5 else None
        Bkn = B.double() if b_layout == "kn" else B.double().t()
        ref = A.double() @ Bkn
        if bias is not None:
            ref = ref + bias.double()
        if act == "gelu":
            ref = F.gelu(ref)
        return dict(inst=dense_instance(M, N, K), A=A, B=B, C=C, C_base=C_base, b_layout=b_layout, bias=bias,
                    act=act, ref=ref, K=K, keep=(A_base, B_base, C_base),
                    name=f"dense M{M} N{N} K{K} {b_layout} {out_dtype} bias={bias is not None} {act}")
    b = rng.choice([64, 384, 1024])
    T = rng.randint(1, 512)
    kind = rng.choice(["scores", "context"])
    M, N, K, dyn, b_layout = (T, T, 64, ("i", "j"), "nk") if kind == "scores" else (T, 64, T, ("i", "k"), "kn")
    out_dtype = torch.float32 if rng.random() < 0.15 else torch.bfloat16
    A_base, A = _padded((b, M, K), torch.bfloat16, dev, g)
    B_base, B = _padded((b, K, N) if b_layout == "kn" else (b, N, K), torch.bfloat16, dev, g)
    C_base, C = _padded((b, M, N), out_dtype, dev, g, fill=float("nan"))
    Bkn = B.double() if b_layout == "kn" else B.double().transpose(1, 2)
    return dict(inst=bmm_instance(b, M, N, K, dyn), A=A, B=B, C=C, C_base=C_base, b_layout=b_layout, bias=None,
                act=None, ref=A.double() @ Bkn, K=K, keep=(A_base, B_base, C_base),
                name=f"bmm {kind} b{b} T{T} {b_layout} {out_dtype}")


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_random_large_problems_alone_and_grouped(cuda, seed):
    rng = random.Random(seed)
    g = torch.Generator(device="cpu").manual_seed(seed)
    probs = [_draw_large(rng, g, cuda) for _ in range(8)]
    recs = Planner().plan([p["inst"] for p in probs])
    for p, r in zip(probs, recs):
        ex = Executable([gemm_desc(p["A"], p["B"], p["C"], p["b_layout"], bias=p["bias"], activation=p["act"])],
                        [r.program], p["keep"])
        ex.launch()
        torch.cuda.synchronize()
        _check(p, "alone")
        ex.close()
    for p in probs:
        p["C_base"].fill_(float("nan"))
    descs = [gemm_desc(p["A"], p["B"], p["C"], p["b_layout"], bias=p["bias"], activation=p["act"]) for p in probs]
    ex = Executable(descs, [r.program for r in recs], [t for p in probs for t in p["keep"]])
    ex.launch()
    torch.cuda.synchronize()
    for p in probs:
        _check(p, "grouped")
    ex.close()
