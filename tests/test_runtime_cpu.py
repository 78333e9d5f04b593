"""Runtime planner (ftb_plan_batch) on CPU: B200-mode plans lower to tables
that tile C exactly once; the fallback ladder covers shapes the strict
legality cannot; parity-mode Top-1 equals the facade's (reference-exact)
ranking; the plan cache round-trips."""

import numpy as np
import pytest

from paper_2407_21418_b200 import _lib
from paper_2407_21418_b200.execute import lower_table
from paper_2407_21418_b200.mktune.filtering import compile_shape
from paper_2407_21418_b200.mktune.hardware import b200_bf16
from paper_2407_21418_b200.mktune.scoring import rank_topk
from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance


def desc_for(inst):
    e = inst.extents
    d = _lib.GemmDesc()
    if "b" in e:
        d.op, d.batch, d.M, d.N, d.K = _lib.OP_BMM, e["b"], e["i"], e["j"], e["k"]
    else:
        d.op, d.batch, d.M, d.N, d.K = _lib.OP_DENSE, 1, e["i"], e["j"], e["k"]
    d.A = d.B = d.C = 256
    d.lda = d.ldb = (d.K + 7) // 8 * 8
    d.ldc = d.N
    d.a_batch_stride, d.b_batch_stride, d.c_batch_stride = d.M * d.lda, d.N * d.ldb, d.M * d.N
    d.b_layout, d.in_dtype, d.out_dtype, d.orientation = _lib.B_NK, _lib.DT_BF16, _lib.DT_BF16, -1
    return d


def covered_once(table, d):
    cov = np.zeros((d.batch, d.M, d.N), dtype=np.int32)
    swap_guess = []
    for _, b, l0, c0, ll, cl, nm, _ in table:
        swap_guess.append((b, l0, c0, ll, cl))
    # orientation is per problem: try both and accept the one that tiles exactly
    for swap in (False, True):
        cov[:] = 0
        ok = True
        for b, l0, c0, ll, cl in swap_guess:
            if swap:
                if c0 + cl > d.M or l0 + ll > d.N:
                    ok = False
                    break
                cov[b, c0:c0 + cl, l0:l0 + ll] += 1
            else:
                if l0 + ll > d.M or c0 + cl > d.N:
                    ok = False
                    break
                cov[b, l0:l0 + ll, c0:c0 + cl] += 1
        if ok and (cov == 1).all():
            return True
    return False


SHAPES = [dense_instance(160, 2304, 768), dense_instance(1216, 768, 768), dense_instance(2116, 768, 768),
          dense_instance(1, 4096, 4096), dense_instance(8191, 4096, 4096), bmm_instance(384, 38, 38, 64),
          bmm_instance(384, 62, 64, 62, ("i", "k")), bmm_instance(64, 257, 257, 64)]


@pytest.fixture(scope="module")
def planned():
    pl = Planner(threads=4)
    return pl, pl.plan(SHAPES)


@pytest.mark.parametrize("idx", range(len(SHAPES)))
def test_b200_plans_lower_and_cover(planned, idx):
    _, recs = planned
    inst = SHAPES[idx]
    d = desc_for(inst)
    table, info = lower_table([d], [recs[idx].program])
    assert covered_once(table, d)
    assert info.true_out == d.batch * d.M * d.N


def test_fallback_ladder_reports_rung(planned):
    _, recs = planned
    r = recs[2]  # Dense M=2116: strict tcgen05 tiles are multiples of 32 and cannot cover 2116 exactly
    assert r.stage >= 4
    assert r.describe()["fallback_stage"] == r.stage


def test_parity_mode_top1_equals_facade():
    hw = b200_bf16(tcgen05=False)
    pl = Planner(hw=hw, threads=2)
    for inst in (dense_instance(53, 768, 768), dense_instance(160, 2304, 768), bmm_instance(384, 38, 38, 64)):
        rec = pl.plan([inst])[0]
        res = compile_shape(inst, hw)
        top = rank_topk(res.candidates, inst, k=1)[0]
        spec = inst.spec
        axes = tuple(spec.space_axes) + tuple(spec.reduce_axes)
        g = rec.program
        got = [([int(g.smem[p][a]) for a in range(len(axes))], int(g.count[p])) for p in range(g.n_parts)]
        want = [([k.smem_tile[a] for a in axes], n) for k, n in top.parts]
        assert got == want
        assert g.sia == top.sia


def test_plan_cache_roundtrip(planned, tmp_path):
    pl, recs = planned
    f = tmp_path / "plans.json"
    pl.save(f)
    pl2 = Planner(threads=1)
    assert pl2.load(f) == len(SHAPES)
    again = pl2.plan(SHAPES)
    for a, b in zip(recs, again):
        assert a.describe()["parts"] == b.describe()["parts"]


def test_gemm_desc_rejects_operands_that_disagree():
    """the TMA descriptors and the work table are built from these
    extents, so B's K / batch and C's shape must agree with A (checked before
    anything touches a device; CPU tensors suffice)."""
    import pytest
    import torch

    from paper_2407_21418_b200.execute import gemm_desc

    bf = torch.bfloat16
    A = torch.zeros(16, 64, dtype=bf)
    with pytest.raises(ValueError, match="inner dimensions"):
        gemm_desc(A, torch.zeros(32, 128, dtype=bf), torch.zeros(16, 128, dtype=bf), "kn")   # B has K = 32
    with pytest.raises(ValueError, match="inner dimensions"):
        gemm_desc(A, torch.zeros(128, 32, dtype=bf), torch.zeros(16, 128, dtype=bf), "nk")   # B^T has K = 32
    with pytest.raises(ValueError, match="C has shape"):
        gemm_desc(A, torch.zeros(64, 128, dtype=bf), torch.zeros(16, 100, dtype=bf), "kn")
    with pytest.raises(ValueError, match="Dense needs"):
        gemm_desc(A, torch.zeros(2, 64, 128, dtype=bf), torch.zeros(16, 128, dtype=bf), "kn")
    A3 = torch.zeros(4, 16, 64, dtype=bf)
    with pytest.raises(ValueError, match="B has batch"):
        gemm_desc(A3, torch.zeros(3, 64, 32, dtype=bf), torch.zeros(4, 16, 32, dtype=bf), "kn")
    with pytest.raises(ValueError, match="C has shape"):
        gemm_desc(A3, torch.zeros(4, 64, 32, dtype=bf), torch.zeros(4, 16, 31, dtype=bf), "kn")
    with pytest.raises(ValueError, match="b_layout"):
        gemm_desc(A, torch.zeros(64, 128, dtype=bf), torch.zeros(16, 128, dtype=bf), "xx")
    with pytest.raises(ValueError, match="CUDA tensor"):  # consistent shapes reach the device check
        gemm_desc(A, torch.zeros(64, 128, dtype=bf), torch.zeros(16, 128, dtype=bf), "kn")


def test_plan_cache_key_covers_the_whole_descriptor():
    """Two descriptors with the same name but different tcgen05 fields must
    not share plan-cache entries (runtime.Planner keys on the full doc)."""
    import dataclasses

    from paper_2407_21418_b200.mktune.hardware import b200_bf16
    from paper_2407_21418_b200.runtime import Planner, dense_instance

    base = b200_bf16(tcgen05=True)
    a, b = Planner(hw=base), Planner(hw=dataclasses.replace(base, mma_n_max=128, tmem_columns=256))
    inst = dense_instance(1216, 2304, 768)
    assert a._key(inst) != b._key(inst)
    assert a._key(inst) == Planner(hw=base)._key(inst)
