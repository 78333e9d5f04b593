"""torch.library ops (SURVEY §8(b) PyTorch wrapper): fake kernels give the
right shapes/dtypes on meta tensors (CPU), CPU inputs are refused loudly
(no CPU path), and on a B200 the ops match float64 references, including
non-TMA-legal strides and one grouped execute_table launch."""

import pytest
import torch

import paper_2407_21418_b200.torch_ops  # noqa: F401  (registers torch.ops.ftb.*)


def test_fake_kernels_shapes_on_meta():
    bf = torch.bfloat16
    A = torch.empty(37, 768, device="meta", dtype=bf)
    assert torch.ops.ftb.dense(A, torch.empty(2304, 768, device="meta", dtype=bf), "nk", None, "none").shape == (37, 2304)
    assert torch.ops.ftb.dense(A, torch.empty(768, 100, device="meta", dtype=bf), "kn", None, "gelu").shape == (37, 100)
    f32 = torch.ops.ftb.dense(torch.empty(5, 64, device="meta"), torch.empty(64, 8, device="meta"), "kn", None, "none")
    assert f32.dtype == torch.float32 and f32.shape == (5, 8)
    Q = torch.empty(384, 38, 64, device="meta", dtype=bf)
    assert torch.ops.ftb.bmm(Q, torch.empty(384, 38, 64, device="meta", dtype=bf), "nk", "ij").shape == (384, 38, 38)
    outs = torch.ops.ftb.execute_table([A, Q], [torch.empty(768, 64, device="meta", dtype=bf),
                                                torch.empty(384, 64, 50, device="meta", dtype=bf)], "kn,kn")
    assert [tuple(o.shape) for o in outs] == [(37, 64), (384, 38, 50)]


def test_cpu_inputs_are_refused():
    with pytest.raises(RuntimeError, match="CUDA"):
        torch.ops.ftb.dense(torch.ones(4, 8, dtype=torch.bfloat16), torch.ones(8, 8, dtype=torch.bfloat16), "kn",
                            None, "none")


@pytest.mark.gpu
def test_dense_bmm_and_table_on_gpu(cuda):
    from _numerics import assert_close

    g = torch.Generator(device="cpu").manual_seed(5)

    def rnd(*s, dtype=torch.bfloat16):
        return (torch.rand(*s, generator=g) * 2 - 1).to(dtype).to(cuda)

    A, W, b = rnd(130, 100), rnd(300, 100), rnd(300)  # K=100: row stride not a multiple of 8 -> repacked
    C = torch.ops.ftb.dense(A, W, "nk", b, "gelu")
    ref = torch.nn.functional.gelu(A.double() @ W.double().t() + b.double())
    assert_close(C, ref, 100, "dense", scale=1.2)
    Q, K = rnd(12, 45, 64), rnd(12, 45, 64)
    S = torch.ops.ftb.bmm(Q, K, "nk", "ij")
    ref = Q.double() @ K.double().transpose(1, 2)
    assert_close(S, ref, 64, "bmm")
    As, Bs, lays = [A, Q, rnd(7, 768)], [W, K, rnd(768, 256)], ["nk", "nk", "kn"]
    outs = torch.ops.ftb.execute_table(As, Bs, ",".join(lays))
    for a, bb, lay, o in zip(As, Bs, lays, outs):
        bk = bb.double() if lay == "kn" else bb.double().transpose(-1, -2)
        r = a.double() @ bk
        assert_close(o, r, a.shape[-1], "execute_table")
    torch.library.opcheck(torch.ops.ftb.dense.default, (A, W, "nk", b, "gelu"),
                          test_utils=("test_schema", "test_faketensor"))
