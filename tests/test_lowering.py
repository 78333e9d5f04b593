"""Host-only lowering (ftb_lower): every uKernel rectangle of a plan becomes
MMA-sized work items that tile C exactly once; validation rejects plans
that do not cover tau (combine.py:189-193)."""

import numpy as np
import pytest

from paper_2407_21418_b200 import _lib
from paper_2407_21418_b200.execute import lower_table, program_struct
from paper_2407_21418_b200.mktune import errors


def desc(op, batch, M, N, K, b_layout=_lib.B_NK, dt=_lib.DT_BF16, orientation=-1):
    d = _lib.GemmDesc()
    d.op, d.batch, d.M, d.N, d.K = op, batch, M, N, K
    d.A = d.B = d.C = 256
    d.lda = d.ldb = ((K + 7) // 8) * 8
    if b_layout == _lib.B_KN:
        d.ldb = ((N + 7) // 8) * 8
    d.ldc = N
    d.a_batch_stride, d.b_batch_stride, d.c_batch_stride = M * d.lda, N * K, M * N
    d.b_layout, d.in_dtype, d.out_dtype, d.orientation = b_layout, dt, dt, orientation
    return d


def _unused_coverage(table, d):
    cov = np.zeros((d.batch, d.M, d.N), dtype=np.int32)
    for w in table:
        _, b, l0, c0, ll, cl, nm, _ = w
        assert ll <= 128 and cl <= 256 and nm >= cl
        if d.__dict__ if False else None:
            pass
    return cov


def apply(table, d, swap):
    cov = np.zeros((d.batch, d.M, d.N), dtype=np.int32)
    for _, b, l0, c0, ll, cl, nm, _ in table:
        if swap:
            cov[b, c0:c0 + cl, l0:l0 + ll] += 1
        else:
            cov[b, l0:l0 + ll, c0:c0 + cl] += 1
    return cov


@pytest.mark.parametrize("orientation", [0, 1])
@pytest.mark.parametrize("M,N,parts,tau", [
    (200, 320, [((1, 8), (30, 64, 64), 3), ((1, 8), (30, 128, 64), 1)], 1),
    (4096, 768, [((1, 8), (16, 192, 64), 4), ((1, 8), (112, 192, 64), 36)], 0),
    (1, 768, [((1, 1), (1, 64, 64), 12)], 1),
    (509, 768, [((1, 8), (30, 512, 64), 1), ((1, 8), (30, 256, 64), 1)], 1),
])
def test_dense_tiles_cover_once(orientation, M, N, parts, tau):
    d = desc(_lib.OP_DENSE, 1, M, N, 256, orientation=orientation)
    t, info = lower_table([d], [program_struct(2, tau, parts)])
    assert (apply(t, d, orientation == 1) == 1).all()
    assert info.true_out == M * N


def test_bmm_tiles_cover_once():
    d = desc(_lib.OP_BMM, 6, 37, 37, 64)
    t, info = lower_table([d], [program_struct(3, 0, [((1, 1, 1), (2, 37, 64, 64), 3)])])
    assert (apply(t, d, False) == 1).all() or (apply(t, d, True) == 1).all()


def test_rejects_non_covering_plan():
    d = desc(_lib.OP_DENSE, 1, 100, 320, 64)
    with pytest.raises(errors.InputError):
        lower_table([d], [program_struct(2, 1, [((1, 8), (30, 64, 64), 4)])])  # 256 != 320
    with pytest.raises(errors.InputError):
        lower_table([d], [program_struct(2, 1, [((1, 8), (30, 64, 64), 3), ((1, 8), (20, 128, 64), 1)])])


def test_padding_ratio_matches_covered_extents():
    d = desc(_lib.OP_DENSE, 1, 53, 768, 768)
    _, info = lower_table([d], [program_struct(2, 1, [((1, 8), (8, 64, 64), 12)])])
    assert info.covered_out == 56 * 768 and info.true_out == 53 * 768


@pytest.mark.parametrize("T", [129, 200, 228, 300, 520])
@pytest.mark.parametrize("orientation", [0, 1])
def test_mn_major_piece_starts_are_tma_aligned(T, orientation):
    """B as [K, N] (MN-major column/lane operand): every piece along N starts
    on a multiple of 8 elements (16-byte TMA box origin) and the pieces still
    tile C exactly once."""
    d = desc(_lib.OP_BMM, 1, T, T, 64, b_layout=_lib.B_KN, orientation=orientation)
    t, _ = lower_table([d], [program_struct(3, 1, [((1, 1, 1), (1, T, 64 * ((T + 63) // 64), 64), 1)])])
    swap = orientation == 1
    for _, b, l0, c0, ll, cl, nm, _ in t:
        n_start = l0 if swap else c0
        assert n_start % 8 == 0
    assert (apply(t, d, swap) == 1).all()


@pytest.mark.parametrize("b_layout", [_lib.B_NK, _lib.B_KN])
@pytest.mark.parametrize("orientation", [0, 1])
@pytest.mark.parametrize("N", [232, 300, 1000])
def test_output_column_piece_starts_are_tma_aligned(b_layout, orientation, N):
    """Pieces along j (C's innermost dimension) start on multiples of 8 in
    both orientations: TMA store boxes need 16-byte origins."""
    d = desc(_lib.OP_DENSE, 1, 130, N, 256, b_layout=b_layout, orientation=orientation)
    t, _ = lower_table([d], [program_struct(2, 0, [((1, 1), (130, 256, 64), 1)])])
    swap = orientation == 1
    for _, b, l0, c0, ll, cl, nm, _ in t:
        assert (l0 if swap else c0) % 8 == 0
    assert (apply(t, d, swap) == 1).all()


def test_items_rasterised_for_l2_locality():
    """Each problem's items are ordered by column group (~32 MiB of the column
    operand over K: 2048 columns at K = 8192), snake order over lanes between
    groups (exec.cu), and still tile C exactly once."""
    M = N = K = 8192
    d = desc(_lib.OP_DENSE, 1, M, N, K, orientation=0)
    t, _ = lower_table([d], [program_struct(2, 0, [((1, 1), (128, 256, 64), M // 128)])])
    group = (32 << 20) // (K * 2)
    gids = [c0 // group for _, _, l0, c0, *_ in t]
    assert gids == sorted(gids)  # column groups in order
    for g in sorted(set(gids)):
        lanes = [l0 for (_, _, l0, c0, *_), gi in zip(t, gids) if gi == g]
        runs = [lanes[i] for i in range(0, len(lanes), group // 256)]  # one lane value per lane row
        assert runs == sorted(runs, reverse=(g % 2 == 1))  # snake
    assert (apply(t, d, False) == 1).all()
