"""GPU outputs against the ORACLE (oracle/execute_np.execute_plan: the CPU
fp32 restatement of executing a ProgramPlan, walking its uKernel rectangles
— combine.py:40-55 coverage semantics), one test per BASELINE config family:
C0 (fp32 FFMA validation mode), C1 (all six BERT-base GEMMs of one sequence
length as one grouped launch), C2 (BERT-large attention BMM) and C3 (LLM
Dense). Each plan must cover C exactly once (coverage == 1 everywhere) and
the device result must match the oracle per element (tests/_numerics.py,
fp32 mode 1e-5)."""

import numpy as np
import pytest
import torch

from _numerics import assert_close
from oracle.execute_np import execute_plan
from paper_2407_21418_b200.runtime import Planner
from paper_2407_21418_b200.shapeset import ShapeSet
from paper_2407_21418_b200.workloads import Shape, bert_layer_shapes

pytestmark = pytest.mark.gpu


def _oracle(x, rec):
    sh = x.shape
    A = x.A.float().cpu().numpy()
    B = x.B.float().cpu().numpy()
    if sh.b_layout == "nk":
        B = np.swapaxes(B, -1, -2)
    g = rec.program
    space = ["i", "j"] if sh.kind == "dense" else ["b", "i", "j"]
    axes = space + ["k"]
    parts = [({a: int(g.smem[p][d]) for d, a in enumerate(axes)}, int(g.count[p])) for p in range(g.n_parts)]
    ext = {"i": sh.M, "j": sh.N, "b": sh.batch}
    return execute_plan(A, B, ext, space, space[g.tau], parts)


def _check_set(shapes, seed, ffma=False):
    planner = Planner() if not ffma else Planner(hw=__import__(
        "paper_2407_21418_b200.mktune.hardware", fromlist=["b200_ffma"]).b200_ffma())
    ss = ShapeSet(shapes, planner, device="cuda:0", seed=seed)
    for x in ss.bound:
        x.C_store.fill_(float("nan"))
    ss.launch()
    torch.cuda.synchronize()
    for x, rec in zip(ss.bound, ss.records):
        ref, cov = _oracle(x, rec)
        assert (cov == 1).all(), f"{x.shape}: plan does not cover C exactly once"
        assert_close(x.C, torch.from_numpy(ref), x.shape.K, str(x.shape), ffma=ffma)


def test_c0_ffma_against_oracle(cuda):
    _check_set([Shape("dense", "dense", 1, m, 768, 768, "kn", ("i",), 4, 4) for m in (1, 53, 509)], 0, ffma=True)


def test_c1_bert_layer_against_oracle(cuda):
    _check_set(bert_layer_shapes(38), 1)


def test_c2_attention_against_oracle(cuda):
    _check_set([Shape("bmm", "scores", 1024, T, T, 64, "nk", ("i", "j")) for T in (1, 64, 257)]
               + [Shape("bmm", "context", 1024, T, 64, T, "kn", ("i", "k")) for T in (1, 64, 257)], 2)


def test_c3_llm_dense_against_oracle(cuda):
    _check_set([Shape("dense", "llm", 1, m, 4096, 4096, "nk") for m in (1, 127, 1000)], 3)
