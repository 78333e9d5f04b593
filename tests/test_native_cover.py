"""The runtime planner's last fallback rung (beyond the reference): shapes
whose uKernel candidates admit no exact cover of the composition axis
(combine.py:183-188 raises EmptyResultError for them, and so does the mktune
facade) get an executor-native exact cover. Host-only lowering checks that
every output element is covered exactly once. CPU only."""

import numpy as np
import pytest

from paper_2407_21418_b200 import _lib
from paper_2407_21418_b200.execute import lower_table
from paper_2407_21418_b200.mktune import errors
from paper_2407_21418_b200.mktune.filtering import compile_shape
from paper_2407_21418_b200.mktune.hardware import b200_bf16
from paper_2407_21418_b200.mktune.scoring import rank_topk
from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance

CASES = [  # (kind, b, M, N, K, needs native cover)
    ("bmm", 3, 100, 152, 77, True),     # main axis j = 152: no sum of 64-multiples
    ("bmm", 40, 250, 300, 7, True),
    ("dense", 1, 300, 1000, 100, True),  # neither output axis has a 64-multiple cover
    ("dense", 1, 1, 1000, 5, False),     # covered by the C++ ladder (i as the composition axis)
    ("dense", 1, 129, 200, 40, False),
]


def _inst(kind, b, M, N, K, native=None):
    return bmm_instance(b, M, N, K) if kind == "bmm" else dense_instance(M, N, K)


def _desc(kind, b, M, N, K, native=None):
    d = _lib.GemmDesc()
    d.op = _lib.OP_BMM if kind == "bmm" else _lib.OP_DENSE
    d.batch, d.M, d.N, d.K = b, M, N, K
    d.A = d.B = d.C = 256
    d.lda = d.ldb = (K + 7) // 8 * 8
    d.ldc = (N + 7) // 8 * 8
    d.a_batch_stride, d.b_batch_stride, d.c_batch_stride = M * d.lda, N * d.ldb, M * d.ldc
    if kind == "dense":
        d.a_batch_stride = d.b_batch_stride = d.c_batch_stride = 0
    d.b_layout, d.in_dtype, d.out_dtype, d.orientation = _lib.B_NK, _lib.DT_BF16, _lib.DT_BF16, 0
    return d


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(map(str, c)))
def test_native_cover_plans_and_lowers_exactly(case):
    kind, b, M, N, K, native = case
    rec = Planner().plan([_inst(*case)])[0]
    assert (rec.relaxation == "native-cover" and rec.stage == -1) == native
    table, info = lower_table([_desc(*case)], [rec.program])
    cov = np.zeros((b, M, N), dtype=np.int32)
    for _, bb, l0, c0, ll, cl, _, _ in table:  # orientation 0: lanes = rows of C
        cov[bb, l0:l0 + ll, c0:c0 + cl] += 1
    assert (cov == 1).all()
    assert info.true_flops == 2 * b * M * N * K


def test_reference_semantics_kept_in_facade_and_switch(monkeypatch):
    """The mktune facade (parity API) still raises like the reference, and
    FTB_NATIVE_COVER=0 restores the error in the runtime planner too."""
    inst = _inst(*CASES[0])
    with pytest.raises(errors.EmptyResultError):
        rank_topk(compile_shape(inst, b200_bf16(tcgen05=True)).candidates, inst, k=1)
    monkeypatch.setenv("FTB_NATIVE_COVER", "0")
    with pytest.raises(errors.EmptyResultError):
        Planner().plan([inst])
