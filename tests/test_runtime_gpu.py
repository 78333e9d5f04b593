"""Planner -> lowering -> sm_100a executor, end to end on B200, for every
BASELINE config family: C0 (fp32 FFMA validation mode, 1e-5), C1/C3 Dense,
C2 attention BMM (bf16, 2e-2), and the grouped C1 shape set in one launch.
Reference: the same op in float64 on the device, checked per element
(tests/_numerics.py: 8e-3 relative + sqrt(K)-scaled accumulation term; the
fp32 FFMA mode 1e-5 relative)."""

import pytest
import torch
from _numerics import assert_close

from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import Shape, c1_shapes

pytestmark = pytest.mark.gpu


def close(c, ref, K, what="", **kw):
    """Per-element check (tests/_numerics.py)."""
    assert_close(c, ref, K, what=str(what), **kw)
    return True


@pytest.fixture(scope="module")
def planner():
    return Planner()


@pytest.mark.parametrize("M", [1, 7, 16, 127, 1000, 2116, 4097])
def test_c3_dense_4096(cuda, planner, M):
    g = torch.Generator(device=cuda).manual_seed(M)
    A = (torch.rand(M, 4096, device=cuda, generator=g) * 2 - 1).bfloat16()
    W = (torch.rand(4096, 4096, device=cuda, generator=g) * 2 - 1).bfloat16()
    C = planner.dense(A, W, b_layout="nk")
    torch.cuda.synchronize()
    assert close(C, A.double() @ W.double().t(), 4096)


@pytest.mark.parametrize("M", [1, 2, 53, 64, 127, 509, 512])
def test_c0_fp32_ffma(cuda, planner, M):
    g = torch.Generator(device=cuda).manual_seed(M)
    A = torch.rand(M, 768, device=cuda, generator=g) * 2 - 1
    B = torch.rand(768, 768, device=cuda, generator=g) * 2 - 1
    C = planner.dense(A, B, b_layout="kn")
    torch.cuda.synchronize()
    assert C.dtype == torch.float32
    assert close(C, A.double() @ B.double(), 768, ffma=True)


@pytest.mark.parametrize("T", [1, 8, 64, 257, 512])
def test_c2_bmm_attention(cuda, planner, T):
    shapes = [Shape("bmm", "scores", 1024, T, T, 64, "nk", ("i", "j")),
              Shape("bmm", "context", 1024, T, 64, T, "kn", ("i", "k"))]
    ss = ShapeSet(shapes, planner, device=cuda, seed=T)
    ss.launch()
    torch.cuda.synchronize()
    for i, x in enumerate(ss.bound):
        assert close(x.C, ss.reference_outputs(i), x.shape.K, x.shape)


def test_c1_grouped_table(cuda, planner):
    ss = ShapeSet(c1_shapes(n_draws=4, seed=5), planner, device=cuda, seed=1)
    for x in ss.bound:
        x.C_store.fill_(float("nan"))
    ss.launch()
    torch.cuda.synchronize()
    for i, x in enumerate(ss.bound):
        assert not torch.isnan(x.C.float()).any(), x.shape
        assert close(x.C, ss.reference_outputs(i), x.shape.K, x.shape)


def test_graph_capture_and_replay(cuda, planner):
    ss = ShapeSet(c1_shapes(n_draws=1, seed=2)[:12], planner, device=cuda, seed=2)
    s = torch.cuda.Stream(cuda)
    g = torch.cuda.CUDAGraph()
    ss.launch(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        ss.launch(s)
    for x in ss.bound:
        x.C_store.zero_()
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    for i, x in enumerate(ss.bound):
        assert close(x.C, ss.reference_outputs(i), x.shape.K, x.shape)


def test_e2e_pipelined_round_trip(cuda, planner):
    """Pipelined end-to-end steps (two device buffer sets, overlapped H2D /
    launch / D2H): the host output arena holds every shape's result."""
    ss = ShapeSet(c1_shapes(n_draws=1, seed=3)[:12], planner, device=cuda, seed=3, pinned=True)
    ss.out_arena.fill_(float("nan"))
    ms = ss.e2e_pipelined(3)
    assert ms > 0
    host = ss.host_out_arena.to(cuda)
    ss.launch()
    torch.cuda.synchronize()
    # the last step read back buffer set 0; every output element it holds
    # matches a fresh launch (arena padding stays NaN in both)
    assert torch.allclose(host.float(), ss.out_arena.float(), rtol=0, atol=0, equal_nan=True)
    for i, x in enumerate(ss.bound):
        assert close(x.C, ss.reference_outputs(i), x.shape.K, x.shape)


def test_c4_sweep_sample_one_table(cuda, planner):
    """A sample of the C4 10k-shape sweep (mixed Dense / attention BMM, M and T
    dynamic) planned and executed as ONE table. Size-independent check on every
    shape: row checksums C @ 1 == A @ (B @ 1) in float64 (scaled by the row
    sums of |C|); shapes small enough also get the full element-wise check."""
    from paper_2407_21418_b200.workloads import c4_shapes

    shapes = c4_shapes(48, seed=11)
    ss = ShapeSet(shapes, planner, device=cuda, seed=11)
    ss.out_arena.fill_(float("nan"))
    ss.launch()
    torch.cuda.synchronize()
    for i, x in enumerate(ss.bound):
        C = x.C.double()
        assert not torch.isnan(C).any(), x.shape
        Bkn = x.B.double().transpose(-1, -2) if x.shape.b_layout == "nk" else x.B.double()
        expect = (x.A.double() @ Bkn.sum(-1, keepdim=True)).squeeze(-1)
        err = (C.sum(-1) - expect).abs().max() / C.abs().sum(-1).max().clamp_min(1e-30)
        assert err.item() < 1e-2, x.shape
        if x.shape.flops < 2e9:
            assert close(x.C, ss.reference_outputs(i), x.shape.K, x.shape)


@pytest.mark.parametrize("M", [1, 37, 160, 1024, 2116])
@pytest.mark.parametrize("act", [None, "gelu"])
@pytest.mark.parametrize("bias_dtype", [torch.bfloat16, torch.float32, None])
def test_dense_fused_bias_gelu(cuda, planner, M, act, bias_dtype):
    """f-3: Dense + bias (+ GELU, erf form) fused into the epilogue, on every
    epilogue path (TMA stores, predicated stores, split-K reduction) vs torch."""
    import torch.nn.functional as F

    N, K = 3072, 768
    g = torch.Generator(device=cuda).manual_seed(M)
    A = (torch.rand(M, K, device=cuda, generator=g) * 2 - 1).bfloat16()
    W = (torch.rand(N, K, device=cuda, generator=g) * 2 - 1).bfloat16() * 0.05
    bias = None if bias_dtype is None else (torch.rand(N, device=cuda, generator=g) * 2 - 1).to(bias_dtype)
    C = planner.dense(A, W, b_layout="nk", bias=bias, activation=act)
    torch.cuda.synchronize()
    ref = A.double() @ W.double().t()
    if bias is not None:
        ref = ref + bias.double()
    if act == "gelu":
        ref = F.gelu(ref)
    assert close(C, ref, K, scale=0.05 * 1.2)


def test_fp32_ffma_fused_bias_gelu(cuda, planner):
    import torch.nn.functional as F

    g = torch.Generator(device=cuda).manual_seed(3)
    A = torch.rand(53, 768, device=cuda, generator=g) * 2 - 1
    B = torch.rand(768, 768, device=cuda, generator=g) * 2 - 1
    bias = torch.rand(768, device=cuda, generator=g)
    C = planner.dense(A, B, b_layout="kn", bias=bias, activation="gelu")
    torch.cuda.synchronize()
    assert close(C, F.gelu(A.double() @ B.double() + bias.double()), 768, ffma=True, scale=1.2)


@pytest.mark.parametrize("T", [5, 38, 128])
def test_bert_encoder_layer_module_swap(cuda, planner, T):
    """f-3 module swap: a torch TransformerEncoderLayer (BERT-base layout,
    GELU, post-norm) vs the same layer with its six GEMMs on the executor
    (fused bias / GELU epilogues, attention BMMs batched over heads)."""
    from paper_2407_21418_b200.bert import EncoderLayer

    torch.manual_seed(T)
    layer = torch.nn.TransformerEncoderLayer(768, 12, 3072, dropout=0.0, activation="gelu", batch_first=True,
                                             device=cuda).eval()
    with torch.no_grad():
        for p in layer.parameters():  # bf16-representable weights: the comparison isolates the executor
            p.copy_(p.bfloat16().float())
    x = (torch.randn(4, T, 768, device=cuda)).bfloat16()
    with torch.no_grad():
        ref = layer(x.float())
    ours = EncoderLayer.from_torch(layer, planner)(x)
    torch.cuda.synchronize()
    err = ((ours.float() - ref).abs().max() / ref.abs().max()).item()
    assert err < 3e-2, err


def test_sharded_c4_executor_single_rank(cuda, planner):
    """shard.run_sharded with the GPU executor (world 1): every shape of a C4
    sample executes in grouped chunk launches and its output checksum
    matches the size-independent expectation sum(C) = 1^T A B 1; inputs are
    seeded by global shape index, so a re-run over a different chunking gives
    the identical checksums."""
    import json

    from paper_2407_21418_b200.shard import checksum_ok, make_gpu_executor, run_sharded
    from paper_2407_21418_b200.workloads import c4_shapes

    shapes = c4_shapes(40, seed=5)
    ex = make_gpu_executor(planner, cuda)
    _, merged = run_sharded(shapes, 0, 1, planner, 1.6792e15, execute=ex)
    assert [r.index for r in merged] == list(range(len(shapes)))
    cs = [json.loads(r.checksum) for r in merged]
    assert all(checksum_ok(c) for c in cs), [c for c in cs if not checksum_ok(c)][:3]
    ex2 = make_gpu_executor(planner, cuda, max_chunk_bytes=2e8)
    _, merged2 = run_sharded(shapes, 0, 1, planner, 1.6792e15, execute=ex2)
    assert ex2.stats["chunks"] > ex.stats["chunks"]
    assert [r.checksum for r in merged2] == [r.checksum for r in merged]


def test_captured_table_survives_destroy(cuda):
    """A table launched inside a CUDA-graph capture stays valid for the
    graph after its handle is destroyed (the runtime's table LRU may evict it
    at any time): replays after close() still compute the right result."""
    from paper_2407_21418_b200.execute import Executable, gemm_desc
    from paper_2407_21418_b200.runtime import Planner, dense_instance

    g = torch.Generator(device="cpu").manual_seed(2)
    A = (torch.rand(300, 768, generator=g) * 2 - 1).bfloat16().to(cuda)
    W = (torch.rand(768, 768, generator=g) * 2 - 1).bfloat16().to(cuda)
    C = torch.empty(300, 768, dtype=torch.bfloat16, device=cuda)
    ex = Executable([gemm_desc(A, W, C, "nk")], [Planner().plan([dense_instance(300, 768, 768)])[0].program])
    s = torch.cuda.Stream(cuda)
    ex.launch(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        ex.launch(s)
    ex.close()
    for _ in range(3):  # churn the pool with other tables
        Executable([gemm_desc(A, W, C, "nk")], [Planner().plan([dense_instance(300, 768, 768)])[0].program]).close()
    C.zero_()
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    assert close(C, A.double() @ W.double().t(), 768, "replay after close")


def test_table_churn_create_launch_destroy(cuda):
    """The table allocator under churn: hundreds of tables of random shapes
    created (async upload through the pinned staging pool), launched on two
    streams and destroyed right away (stream-ordered free) — every output
    correct, no device-wide synchronisation needed."""
    import random

    from paper_2407_21418_b200.execute import Executable, gemm_desc
    from paper_2407_21418_b200.runtime import Planner, dense_instance

    rng = random.Random(4)
    planner = Planner()
    streams = [torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)]
    jobs = []
    for i in range(120):
        M, N, K = rng.randint(1, 700), rng.choice([64, 256, 768, 1000]), rng.choice([64, 256, 768])
        A = (torch.rand(M, K, device=cuda) * 2 - 1).bfloat16()
        W = (torch.rand(N, K, device=cuda) * 2 - 1).bfloat16()
        C = torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda)
        ex = Executable([gemm_desc(A, W, C, "nk")], [planner.plan([dense_instance(M, N, K)])[0].program])
        s = streams[i % 2]
        s.wait_stream(torch.cuda.current_stream(cuda))  # inputs were written on the current stream
        ex.launch(s)
        ex.close()  # freed in stream order after its launch
        jobs.append((A, W, C, K))
    torch.cuda.synchronize()
    for A, W, C, K in jobs:
        assert close(C, A.double() @ W.double().t(), K, "churn")


def test_tables_created_inside_a_torch_graph_capture(cuda, planner):
    """A GEMM whose output is allocated inside torch.cuda.graph (the graph's
    private pool: new addresses, so a new table) builds its table mid-capture
    (relaxed capture mode for the table's own allocation and upload) and the
    replayed graph computes the same result as eager execution."""
    g0 = torch.Generator(device="cpu").manual_seed(3)
    A = (torch.rand(96, 256, generator=g0) * 2 - 1).bfloat16().to(cuda)
    W = (torch.rand(384, 256, generator=g0) * 2 - 1).bfloat16().to(cuda)
    eager = planner.dense(A, W, b_layout="nk")
    s = torch.cuda.Stream(cuda)
    s.wait_stream(torch.cuda.current_stream(cuda))
    with torch.cuda.stream(s):
        planner.dense(A, W, b_layout="nk")
    torch.cuda.current_stream(cuda).wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = planner.dense(A, W, b_layout="nk")
        out2 = torch.relu(out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    assert torch.equal(out2, torch.relu(eager))
