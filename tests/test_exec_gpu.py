"""Executor numerics on B200: hand-built plans of every shape class vs a
plain fp32 reference of the same op (norm-wise relative error)."""

import pytest
import torch

from _numerics import assert_close
from paper_2407_21418_b200.execute import Executable, gemm_desc, program_struct

pytestmark = pytest.mark.gpu

def _ok(c, ref, K, **kw):
    """Per-element check (tests/_numerics.py: 8e-3 relative + an accumulation
    term scaled by sqrt(K); fp32 paths 1e-5)."""
    assert_close(c, ref, K, **kw)
    return True


def _dense(M, N, K, b_layout, dtype, dev, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    A = (torch.rand(M, K, generator=g) * 2 - 1).to(dtype).to(dev)
    Bkn = (torch.rand(K, N, generator=g) * 2 - 1).to(dtype).to(dev)
    B = Bkn if b_layout == "kn" else Bkn.t().contiguous()
    ref = A.double() @ Bkn.double()
    return A, B, ref


DENSE_CASES = [
    # (M, N, K, tau, parts[(reg, smem, count)])
    (256, 512, 256, 1, [((1, 8), (128, 128, 64), 4)]),
    (200, 320, 200, 1, [((1, 8), (30, 64, 64), 3), ((1, 8), (30, 128, 64), 1)]),
    (5, 768, 768, 1, [((1, 8), (8, 64, 64), 12)]),
    (1, 768, 768, 1, [((1, 1), (1, 64, 64), 12)]),
    (509, 768, 768, 1, [((1, 8), (30, 32 * 2, 64), 12)]),
    (4096, 1024, 512, 0, [((1, 8), (128, 256, 64), 32)]),
    (1696, 2304, 768, 1, [((1, 8), (106, 128, 64), 18)]),
    (300, 256, 72, 0, [((2, 8), (100, 256, 64), 3)]),
]


@pytest.mark.parametrize("case", DENSE_CASES, ids=lambda c: f"M{c[0]}N{c[1]}K{c[2]}")
@pytest.mark.parametrize("b_layout", ["kn", "nk"])
@pytest.mark.parametrize("orientation", [-1, 0, 1])
def test_dense_bf16(cuda, case, b_layout, orientation):
    M, N, K, tau, parts = case
    A, B, ref = _dense(M, N, K, b_layout, torch.bfloat16, cuda)
    Cout = torch.empty(M, N, dtype=torch.bfloat16, device=cuda)
    Cout.fill_(float("nan"))
    ex = Executable([gemm_desc(A, B, Cout, b_layout, orientation)], [program_struct(2, tau, parts)])
    ex.launch()
    torch.cuda.synchronize()
    assert not torch.isnan(Cout.float()).any(), "uncovered output elements"
    assert _ok(Cout, ref, K)


@pytest.mark.parametrize("case", DENSE_CASES, ids=lambda c: f"M{c[0]}N{c[1]}K{c[2]}")
@pytest.mark.parametrize("b_layout", ["kn", "nk"])
@pytest.mark.parametrize("mode", ["pair", "no_tma_store", "no_splitk"])
def test_dense_bf16_kernel_modes(cuda, case, b_layout, mode, monkeypatch):
    """The CTA-pair kernel (FTB_PAIR=1), the predicated st.global epilogue
    (FTB_TMA_STORE=0) and the unsplit K loop (FTB_SPLITK=0; small tables split
    K by default) against the same reference as the default path."""
    if mode == "pair":
        monkeypatch.setenv("FTB_PAIR", "1")
    elif mode == "no_tma_store":
        monkeypatch.setenv("FTB_TMA_STORE", "0")
    else:
        monkeypatch.setenv("FTB_SPLITK", "0")
    M, N, K, tau, parts = case
    A, B, ref = _dense(M, N, K, b_layout, torch.bfloat16, cuda, seed=5)
    Cout = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda)
    ex = Executable([gemm_desc(A, B, Cout, b_layout)], [program_struct(2, tau, parts)])
    ex.launch()
    torch.cuda.synchronize()
    assert not torch.isnan(Cout.float()).any(), "uncovered output elements"
    assert _ok(Cout, ref, K)


@pytest.mark.parametrize("orientation", [0, 1])
@pytest.mark.parametrize("N", [100, 104, 99])
def test_dense_strided_output_untouched_padding(cuda, orientation, N):
    """C as a view of a wider buffer: nothing may be written past the tensor
    edge (N) — TMA-store boxes clip at 16 B, so N % 8 != 0 takes the
    predicated epilogue."""
    M, K = 200, 128
    A, B, ref = _dense(M, N, K, "nk", torch.bfloat16, cuda, seed=7)
    store = torch.full((M, 136), float("nan"), dtype=torch.bfloat16, device=cuda)
    Cout = store[:, :N]
    ex = Executable([gemm_desc(A, B, Cout, "nk", orientation)], [program_struct(2, 0, [((1, 1), (200, N, 64), 1)])])
    ex.launch()
    torch.cuda.synchronize()
    assert torch.isnan(store[:, N:].float()).all(), "store wrote past the tensor edge"
    assert _ok(Cout, ref, K)


@pytest.mark.parametrize("b_layout", ["kn", "nk"])
def test_dense_f32_out(cuda, b_layout):
    M, N, K = 130, 384, 192
    A, B, ref = _dense(M, N, K, b_layout, torch.bfloat16, cuda, seed=3)
    Cout = torch.full((M, N), float("nan"), dtype=torch.float32, device=cuda)
    ex = Executable([gemm_desc(A, B, Cout, b_layout)], [program_struct(2, 1, [((1, 8), (65, 128, 64), 3)])])
    ex.launch()
    torch.cuda.synchronize()
    assert _ok(Cout, ref, K)


@pytest.mark.parametrize("T", [1, 5, 37, 64, 128])
@pytest.mark.parametrize("kind", ["scores", "context"])
@pytest.mark.parametrize("b,pack", [(6, True), (9, True), (6, False)])
def test_bmm_bf16(cuda, T, kind, b, pack, monkeypatch):
    """BMM attention shapes; with packing, up to 4 consecutive batch entries
    share one work item and one 3-D TMA box per operand (last group ragged)."""
    if not pack:
        monkeypatch.setenv("FTB_NO_PACK", "1")
    g = torch.Generator().manual_seed(T)
    if kind == "scores":
        # Q [b,T,64] @ K^T: B given as K [b, T(j), 64(k)] -> "nk" layout
        M, N, Kd, layout = T, T, 64, "nk"
    else:
        # P [b,T,T] @ V [b,T(k),64(j)] -> "kn" layout; P row stride padded to 8
        M, N, Kd, layout = T, 64, T, "kn"
    ldk = (Kd + 7) // 8 * 8
    Abuf = torch.zeros(b, M, ldk, dtype=torch.bfloat16)
    Abuf[:, :, :Kd] = (torch.rand(b, M, Kd, generator=g) * 2 - 1).to(torch.bfloat16)
    A = Abuf.to(cuda)[:, :, :Kd]
    if layout == "nk":
        Bt = (torch.rand(b, N, Kd, generator=g) * 2 - 1).to(torch.bfloat16).to(cuda)
        Bkn = Bt.transpose(1, 2)
        B = Bt
    else:
        B = (torch.rand(b, Kd, N, generator=g) * 2 - 1).to(torch.bfloat16).to(cuda)
        Bkn = B
    ref = A.double() @ Bkn.double()
    Cout = torch.full((b, M, N), float("nan"), dtype=torch.bfloat16, device=cuda)
    jt = ((N + 63) // 64) * 64
    parts = [((1, 1, 1), (1, M, jt, 64), b)]  # tau = b, one batch entry per uKernel
    ex = Executable([gemm_desc(A, B, Cout, layout)], [program_struct(3, 0, parts)])
    ex.launch()
    torch.cuda.synchronize()
    assert not torch.isnan(Cout.float()).any()
    assert _ok(Cout, ref, Kd)


def test_grouped_launch(cuda):
    """Many problems of different shapes and plans in ONE launch."""
    descs, progs, refs, outs, keep = [], [], [], [], []
    for s, (M, N, K, tau, parts) in enumerate(DENSE_CASES[:6]):
        A, B, ref = _dense(M, N, K, "nk", torch.bfloat16, cuda, seed=10 + s)
        Cout = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda)
        descs.append(gemm_desc(A, B, Cout, "nk"))
        progs.append(program_struct(2, tau, parts))
        refs.append((ref, K))
        outs.append(Cout)
        keep += [A, B, Cout]
    ex = Executable(descs, progs, keep)
    ex.launch()
    torch.cuda.synchronize()
    for c, (r, k) in zip(outs, refs):
        assert _ok(c, r, k)


@pytest.mark.parametrize("M", [1, 53, 509])
@pytest.mark.parametrize("b_layout", ["kn", "nk"])
def test_dense_ffma_fp32(cuda, M, b_layout):
    N = K = 768
    A, B, ref = _dense(M, N, K, b_layout, torch.float32, cuda, seed=M)
    Cout = torch.full((M, N), float("nan"), dtype=torch.float32, device=cuda)
    ex = Executable([gemm_desc(A, B, Cout, b_layout)], [program_struct(2, 1, [((1, 8), (30, 64, 32), 12)])])
    ex.launch()
    torch.cuda.synchronize()
    assert ex.info.kernel == "ffma"
    assert _ok(Cout, ref, K, ffma=True)


def test_split_k_repeated_launches_deterministic(cuda):
    """Split-K counters re-arm themselves: repeated launches (and a CUDA graph
    replay) give bit-identical results (fixed summation order)."""
    M, N, K = 64, 1024, 4096
    A, B, ref = _dense(M, N, K, "nk", torch.bfloat16, cuda, seed=21)
    Cout = torch.empty(M, N, dtype=torch.bfloat16, device=cuda)
    ex = Executable([gemm_desc(A, B, Cout, "nk")], [program_struct(2, 1, [((1, 1), (64, 256, 64), 4)])])
    ex.launch()
    torch.cuda.synchronize()
    first = Cout.clone()
    assert _ok(Cout, ref, K)
    for _ in range(3):
        Cout.zero_()
        ex.launch()
    torch.cuda.synchronize()
    assert torch.equal(Cout, first)


@pytest.mark.parametrize("M,N,K", [(160, 768, 3072), (96, 1000, 2048), (300, 768, 1024)])
def test_column_split_and_split_k_lowerings(cuda, monkeypatch, M, N, K):
    """Under-occupied tables: the column split (256-column items halved) is
    bit-identical to the unsplit lowering, and split-K (parallel rendezvous
    reduction) stays within the bf16 tolerance and is deterministic."""
    A, B, ref = _dense(M, N, K, "nk", torch.bfloat16, cuda, seed=31)
    from paper_2407_21418_b200.runtime import Planner, dense_instance

    prog = Planner().plan([dense_instance(M, N, K)])[0].program
    outs = {}
    for cs, sk in (("0", "0"), ("1", "0"), ("1", "1")):
        monkeypatch.setenv("FTB_COLSPLIT", cs)
        monkeypatch.setenv("FTB_SPLITK", sk)
        Cout = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda)
        ex = Executable([gemm_desc(A, B, Cout, "nk")], [prog])
        for _ in range(3):
            ex.launch()
        torch.cuda.synchronize()
        outs[(cs, sk)] = Cout.clone()
        ex.close()
    assert torch.equal(outs[("0", "0")], outs[("1", "0")])
    assert _ok(outs[("1", "1")], ref, K)


@pytest.mark.parametrize("T", [200, 228, 300])
def test_bmm_kn_layout_split_pieces_tma_aligned(cuda, T):
    """B given as [K, N] makes the column (or, swapped, the lane) operand
    MN-major; the executor's pieces of a > 128-lane / > 256-column rectangle
    must start on multiples of 8 elements (TMA 16-byte box origin). A balanced
    split at 114 or 100 used to fault with an illegal instruction (found by
    tests/test_fuzz_gpu.py)."""
    from paper_2407_21418_b200.runtime import Planner, bmm_instance

    g = torch.Generator(device="cpu").manual_seed(T)
    pad = (T + 7) // 8 * 8
    A = (torch.rand(1, T, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
    B = (torch.rand(1, 64, pad, generator=g) * 2 - 1).bfloat16().to(cuda)[:, :, :T]
    Cb = torch.full((1, T, pad), float("nan"), dtype=torch.bfloat16, device=cuda)
    C = Cb[:, :, :T]
    rec = Planner().plan([bmm_instance(1, T, T, 64)])[0]
    ex = Executable([gemm_desc(A, B, C, "kn")], [rec.program], (A, B, Cb))
    ex.launch()
    torch.cuda.synchronize()
    assert _ok(C, A.double() @ B.double(), 64)
    assert torch.isnan(Cb[:, :, T:].float()).all()


@pytest.mark.parametrize("M", [129, 130, 160])
def test_dense_swap_tma_store_origin_aligned(cuda, M):
    """Swap-AB puts output columns on the lanes: a 232-column rectangle used
    to be cut 116 + 116, giving a TMA store box origin at column 884 (not
    16-byte aligned): illegal instruction (found by tests/test_fuzz_gpu.py)."""
    from paper_2407_21418_b200.runtime import Planner, dense_instance

    N, K = 1000, 256
    A, B, ref = _dense(M, N, K, "nk", torch.bfloat16, cuda, seed=M)
    Cb = torch.full((M, 1008), float("nan"), dtype=torch.bfloat16, device=cuda)
    C = Cb[:, :N]
    rec = Planner().plan([dense_instance(M, N, K)])[0]
    ex = Executable([gemm_desc(A, B, C, "nk", orientation=1)], [rec.program], (A, B, Cb))
    ex.launch()
    torch.cuda.synchronize()
    assert _ok(C, ref, K)
    assert torch.isnan(Cb[:, N:].float()).all()


@pytest.mark.parametrize("M,N,K", [(64, 4096, 4096), (300, 768, 1024), (160, 768, 3072)])
def test_split_k_on_chip_matches_workspace_bitwise(cuda, monkeypatch, M, N, K):
    """Split-K reduced on chip (a cluster of the splits, distributed shared
    memory) and through the global fp32 workspace: each deterministic across
    repeated launches, both within tolerance, and bit-identical whenever both
    use the same split count (same partials, same summation order)."""
    from paper_2407_21418_b200.runtime import Planner, dense_instance

    A, B, ref = _dense(M, N, K, "nk", torch.bfloat16, cuda, seed=41)
    prog = Planner().plan([dense_instance(M, N, K)])[0].program
    outs, ctas = {}, {}
    for cl in ("1", "0"):
        monkeypatch.setenv("FTB_SPLIT_CLUSTER", cl)
        Cout = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda)
        ex = Executable([gemm_desc(A, B, Cout, "nk")], [prog])
        ex.launch()
        torch.cuda.synchronize()
        first = Cout.clone()
        for _ in range(3):
            Cout.fill_(float("nan"))
            ex.launch()
        torch.cuda.synchronize()
        assert torch.equal(Cout, first)
        outs[cl], ctas[cl] = first, ex.info.n_ctas
        ex.close()
    for cl in outs:
        assert _ok(outs[cl], ref, K)
    if ctas["1"] == ctas["0"]:
        assert torch.equal(outs["1"], outs["0"])


@pytest.mark.parametrize("case", ["scores64", "context256", "dense_f32"])
def test_eight_warp_epilogue_bitwise_equal(cuda, monkeypatch, case):
    """The eight-epilogue-warp kernel (two warp groups on alternate items,
    4 KiB staging, half-tile transpose) writes exactly the bits of the common
    kernel: forced on and off over a packed BMM, an unpacked BMM and a Dense
    table with fp32 outputs (predicated store path)."""
    from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance

    g = torch.Generator(device="cpu").manual_seed(7)
    if case == "scores64":
        A = (torch.rand(300, 64, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        B = (torch.rand(300, 64, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        shape, lay, inst, dt = (300, 64, 64), "nk", bmm_instance(300, 64, 64, 64), torch.bfloat16
    elif case == "context256":
        A = (torch.rand(200, 256, 256, generator=g) * 2 - 1).bfloat16().to(cuda)
        B = (torch.rand(200, 256, 72, generator=g) * 2 - 1).bfloat16().to(cuda)[:, :, :70]
        shape, lay, inst, dt = (200, 256, 70), "kn", bmm_instance(200, 256, 70, 256, ("i", "k")), torch.bfloat16
    else:
        A = (torch.rand(3000, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        B = (torch.rand(100, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        shape, lay, inst, dt = (3000, 100), "nk", dense_instance(3000, 100, 64), torch.float32
    prog = Planner().plan([inst])[0].program
    outs = []
    for e8 in ("0", "1"):
        monkeypatch.setenv("FTB_EPI8", e8)
        C = torch.full(shape, float("nan"), dtype=dt, device=cuda)
        ex = Executable([gemm_desc(A, B, C, lay)], [prog])
        ex.launch()
        torch.cuda.synchronize()
        outs.append(C.clone())
        ex.close()
    assert not torch.isnan(outs[0].float()).any()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("case", ["cluster_splitk", "epi8", "common"])
def test_graph_replay_matches_eager_bitwise(cuda, case):
    """CUDA-graph capture and replay (how per-shape timing runs) of each kernel
    instantiation — on-chip split-K cluster, eight-warp epilogue, the common
    kernel — writes exactly the eager launch's bits."""
    from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance

    g = torch.Generator(device="cpu").manual_seed(3)
    if case == "cluster_splitk":
        A = (torch.rand(64, 4096, generator=g) * 2 - 1).bfloat16().to(cuda)
        B = (torch.rand(4096, 4096, generator=g) * 2 - 1).bfloat16().to(cuda)
        shape, lay, inst = (64, 4096), "nk", dense_instance(64, 4096, 4096)
    elif case == "epi8":
        A = (torch.rand(512, 64, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        B = (torch.rand(512, 64, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        shape, lay, inst = (512, 64, 64), "nk", bmm_instance(512, 64, 64, 64)
    else:
        A = (torch.rand(1000, 768, generator=g) * 2 - 1).bfloat16().to(cuda)
        B = (torch.rand(2304, 768, generator=g) * 2 - 1).bfloat16().to(cuda)
        shape, lay, inst = (1000, 2304), "nk", dense_instance(1000, 2304, 768)
    C = torch.full(shape, float("nan"), dtype=torch.bfloat16, device=cuda)
    ex = Executable([gemm_desc(A, B, C, lay)], [Planner().plan([inst])[0].program], (A, B, C))
    ex.launch()
    torch.cuda.synchronize()
    eager = C.clone()
    C.fill_(float("nan"))
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        ex.launch(s)
        ex.launch(s)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert not torch.isnan(eager.float()).any()
    assert torch.equal(C, eager)


@pytest.mark.parametrize("case", ["s5", "s23", "s63", "s95", "s121", "s257", "dense_f32_odd"])
def test_bulk_row_store_bitwise_and_bounds(cuda, monkeypatch, case):
    """kFlagBulkStore (whole compact rows that no TMA map can describe: scores
    with T % 8 != 0, fp32 outputs): the rows are written by a 1-D bulk copy
    staged in C's own byte layout plus element stores for the unaligned head
    and tail. C starts at an odd element offset of a guarded buffer (address
    phase != 0 mod 16): every element of C is written, bit-identical to the
    predicated path, and not one guard element is touched."""
    from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance

    g = torch.Generator(device="cpu").manual_seed(11)
    guard = 37
    if case.startswith("s"):
        T, b = int(case[1:]), (384 if int(case[1:]) < 200 else 40)
        A = (torch.rand(b, T, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        B = (torch.rand(b, T, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        shape, lay, inst, dt = (b, T, T), "nk", bmm_instance(b, T, T, 64), torch.bfloat16
        ref = A.double() @ B.double().transpose(1, 2)
        K = 64
    else:
        A = (torch.rand(3000, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        B = (torch.rand(99, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
        shape, lay, inst, dt = (3000, 99), "nk", dense_instance(3000, 99, 64), torch.float32
        ref = A.double() @ B.double().t()
        K = 64
    prog = Planner().plan([inst])[0].program
    n = 1
    for d in shape:
        n *= d
    outs = []
    for bulk in ("0", "1"):
        monkeypatch.setenv("FTB_BULK_STORE", bulk)
        buf = torch.full((n + 2 * guard + 1,), float("nan"), dtype=dt, device=cuda)
        C = buf[guard + 1: guard + 1 + n].view(shape)
        ex = Executable([gemm_desc(A, B, C, lay)], [prog])
        for _ in range(2):
            ex.launch()
        torch.cuda.synchronize()
        assert torch.isnan(buf[: guard + 1].float()).all() and torch.isnan(buf[guard + 1 + n:].float()).all(), \
            "a store landed outside C"
        assert not torch.isnan(C.float()).any(), "an element of C was not written"
        outs.append(C.clone())
        ex.close()
    assert torch.equal(outs[0], outs[1])
    assert_close(outs[1], ref, K, case)


@pytest.mark.parametrize("T", [9, 23, 50, 57, 60, 95, 121, 127, 255, 257])
def test_tma_tail_store_padded_rows(cuda, monkeypatch, T):
    """kFlagTmaTail: C rows padded to a multiple of 8 (16-B row stride, as the
    attention outputs of the bench are allocated) but N = T % 8 != 0. The TMA
    map ends at N rounded down to 8 and each row's last N % 8 columns are
    element stores: bit-identical to the predicated path (FTB_TMA_TAIL=0),
    every element written, the padding columns untouched."""
    from paper_2407_21418_b200.runtime import Planner, bmm_instance

    g = torch.Generator(device="cpu").manual_seed(T)
    b = 384 if T < 200 else 40
    Tp = (T + 7) // 8 * 8
    A = (torch.rand(b, T, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
    B = (torch.rand(b, T, 64, generator=g) * 2 - 1).bfloat16().to(cuda)
    ref = A.double() @ B.double().transpose(1, 2)
    prog = Planner().plan([bmm_instance(b, T, T, 64)])[0].program
    outs = []
    for tail in ("0", "1"):
        monkeypatch.setenv("FTB_TMA_TAIL", tail)
        buf = torch.full((b, T, Tp), float("nan"), dtype=torch.bfloat16, device=cuda)
        C = buf[:, :, :T]
        ex = Executable([gemm_desc(A, B, C, "nk")], [prog])
        ex.launch()
        ex.launch()
        torch.cuda.synchronize()
        assert torch.isnan(buf[:, :, T:].float()).all(), "a store landed in the row padding"
        assert not torch.isnan(C.float()).any(), "an element of C was not written"
        outs.append(C.clone())
        ex.close()
    assert torch.equal(outs[0], outs[1])
    assert_close(outs[1], ref, 64, f"T={T}")


@pytest.mark.parametrize("M,N,K,grows", [(2144, 2304, 768, True), (1728, 3072, 768, True), (3200, 3072, 768, True),
                                         (2144, 2312, 136, False)])
def test_overflow_split_bitwise(cuda, monkeypatch, M, N, K, grows):
    """Overflow split (exec.cu): a table whose last round holds r <= P / 2
    items cuts those into 64/128-column pieces. Bit-identical to the unsplit
    table (same per-element K order), per-element close to fp64, and the
    table really grows (kernel items > logical items). N = 2312 (not a
    multiple of 8, TMA tail stores): its cheapest, last-round items are the
    8-column edge pieces, already narrow, so nothing is split."""
    from paper_2407_21418_b200.runtime import Planner, dense_instance

    g = torch.Generator(device="cpu").manual_seed(M + N)
    A = (torch.rand(M, K, generator=g) * 2 - 1).bfloat16().to(cuda)
    B = (torch.rand(N, K, generator=g) * 2 - 1).bfloat16().to(cuda)
    ref = A.double() @ B.double().t()
    prog = Planner().plan([dense_instance(M, N, K)])[0].program
    Np = (N + 7) // 8 * 8
    outs, items = [], []
    for ov in ("0", "1"):
        monkeypatch.setenv("FTB_OVERFLOW_SPLIT", ov)
        buf = torch.full((M, Np), float("nan"), dtype=torch.bfloat16, device=cuda)
        C = buf[:, :N]
        ex = Executable([gemm_desc(A, B, C, "nk")], [prog])
        ex.launch()
        torch.cuda.synchronize()
        assert torch.isnan(buf[:, N:].float()).all()
        outs.append(C.clone())
        items.append(ex.config()["n_singles"])
        ex.close()
    assert torch.equal(outs[0], outs[1])
    assert (items[1] > items[0]) == grows, items
    assert_close(outs[1], ref, K, f"M{M} N{N} K{K}")


@pytest.mark.parametrize("M,N,K,compact", [(160, 772, 768, False), (160, 771, 768, True), (352, 2312, 768, False),
                                           (1, 1000, 4096, False)])
@pytest.mark.parametrize("switch", ["FTB_COLSPLIT_MIN=128", "FTB_PARAM_MAPS=0", "FTB_TMA_TAIL=0"])
def test_round2_lowering_switches_bitwise(cuda, monkeypatch, M, N, K, compact, switch):
    """Round-2 lowering paths against their switched-off forms, bit for bit:
    32/64-column pieces of one-wave tables (vs 128), descriptors in the
    kernel parameter (vs the table copy), TMA stores up to N rounded down to
    8 with element tails (vs predicated stores) — on row lengths that are
    not a multiple of 8 (padded and compact C), with the padding / guard
    elements untouched."""
    from paper_2407_21418_b200.runtime import Planner, dense_instance

    g = torch.Generator(device="cpu").manual_seed(M * 7 + N)
    A = (torch.rand(M, K, generator=g) * 2 - 1).bfloat16().to(cuda)
    B = (torch.rand(N, K, generator=g) * 2 - 1).bfloat16().to(cuda)
    ref = A.double() @ B.double().t()
    prog = Planner().plan([dense_instance(M, N, K)])[0].program
    ld = N if compact else (N + 7) // 8 * 8
    key, val = switch.split("=")
    outs = []
    for on in (True, False):
        if on:
            monkeypatch.delenv(key, raising=False)
        else:
            monkeypatch.setenv(key, val)
        buf = torch.full((M * ld + 64,), float("nan"), dtype=torch.bfloat16, device=cuda)
        C = buf[:M * ld].view(M, ld)[:, :N]
        ex = Executable([gemm_desc(A, B, C, "nk")], [prog])
        ex.launch()
        torch.cuda.synchronize()
        assert torch.isnan(buf[M * ld:].float()).all()
        if not compact:
            assert torch.isnan(buf[:M * ld].view(M, ld)[:, N:].float()).all(), "row padding written"
        outs.append(C.clone())
        ex.close()
    assert torch.equal(outs[0], outs[1])
    assert_close(outs[0], ref, K, f"M{M} N{N} K{K}")


@pytest.mark.parametrize("b,M,N,K", [(3, 53, 77, 768), (2, 130, 64, 100)])
def test_ffma_bmm_merged_rectangles(cuda, b, M, N, K):
    """FFMA mode on a batched problem with ragged tiles: the merged-rectangle
    lowering (whole uKernel rectangles per <= 64 x 64 CTA) covers every
    element of every batch entry (per-element fp32 tolerance)."""
    from paper_2407_21418_b200.mktune.hardware import b200_ffma
    from paper_2407_21418_b200.runtime import Planner, bmm_instance

    g = torch.Generator(device="cpu").manual_seed(b * M)
    A = (torch.rand(b, M, K, generator=g) * 2 - 1).to(cuda)
    Bm = (torch.rand(b, K, N, generator=g) * 2 - 1).to(cuda)
    C = torch.full((b, M, N), float("nan"), device=cuda)
    prog = Planner(hw=b200_ffma()).plan([bmm_instance(b, M, N, K)])[0].program
    ex = Executable([gemm_desc(A, Bm, C, "kn")], [prog])
    ex.launch()
    torch.cuda.synchronize()
    assert_close(C, A.double() @ Bm.double(), K, "ffma bmm", ffma=True)
