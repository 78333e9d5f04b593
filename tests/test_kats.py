"""Known-answer tests from SPEC.md (acceptance criteria 1, 2, 4, 5 and the
module examples), against the facade; expected values were produced by the
reference (tests/golden/kats.json)."""

from fractions import Fraction

import pytest

from _helpers import KATS
from paper_2407_21418_b200.mktune import combine, filtering, metrics, ukernel, workload
from paper_2407_21418_b200.mktune.hardware import HardwareDescriptor
from cases import dense_doc


def hw80():
    from _helpers import DESCRIPTORS

    return HardwareDescriptor(**DESCRIPTORS["v100_like"])


def test_combination_exactness_ac1():
    assert combine.combin_search([7, 8], 53) == {((7, 3), (8, 4))}
    assert sorted(combine.combin_search([7, 8], 53)) == [tuple(tuple(p) for p in c) for c in KATS["combin_53_7_8"]]


def test_combination_oracle_ac2():
    for case in KATS["random_cases"]:
        got = combine.combin_search(case["tiles"], case["extent"])
        assert sorted(got) == sorted(tuple(tuple(p) for p in c) for c in case["expected"])


def test_reg_tiles_prime_widening():
    assert ukernel.reg_tile_candidates(53, 8) == KATS["reg_tile_53_8"] == [1, 2, 3, 4, 6, 9, 13, 18, 26, 27, 52, 53, 54]
    assert ukernel.reg_tile_candidates(8) == [1, 2, 4, 8]
    assert ukernel.reg_tile_candidates(1) == [1]


def test_occupancy_ac4():
    spec = workload.parse_workload(dense_doc(1, 64, 4, 8192))
    k = ukernel.UKernel(reg_tile={"i": 1, "j": 1}, smem_tile={"i": 1, "j": 8, "k": 8})
    for n in (80, 81, 160):
        f = metrics.occupancy_metric(k, workload.WorkloadInstance(spec, {"i": n}), hw80())
        assert [f.numerator, f.denominator] == KATS["occupancy_80"][str(n)]
    assert float(Fraction(*KATS["occupancy_80"]["81"])) == pytest.approx(0.50625)


def test_sweep_semantics_ac5():
    import numpy as np

    sw = filtering.SweepParams()
    assert sw.num_steps == 46
    spec = workload.parse_workload(dense_doc(8, 8, 4, 8192))
    inst = workload.WorkloadInstance(spec, {"i": 8})
    cs = ukernel.CandidateSet(inst, hw80(), "j", np.ones((3, 2), dtype=np.int64), np.ones((3, 3), dtype=np.int64))
    # (pad, occ) = (0.60, 0.941), (0.49, 1.0), (0.96, 0.95) injected as exact ratios
    cs.columns.update(pad_num=np.array([60, 49, 96]), pad_den=np.array([100, 100, 100]),
                      blocks=np.array([941, 100, 95]), occ_den=np.array([1000, 100, 100]))
    assert list(filtering.retention_steps(cs, sw)) == [10, 0, 1]


def test_flops_volumes_padding_regs_saturation():
    spec = workload.parse_workload(dense_doc(2304, 768, 4, 8192))
    inst = workload.WorkloadInstance(spec, {"i": 128})
    assert workload.flops(inst) == KATS["flops_128_2304_768"] == 452_984_832
    k = ukernel.UKernel(reg_tile={"i": 1, "j": 8}, smem_tile={"i": 8, "j": 64, "k": 64})
    inst53 = workload.WorkloadInstance(workload.parse_workload(dense_doc(768, 768, 4, 8192)), {"i": 53})
    p = metrics.padding_metric(k, inst53)
    assert [p.numerator, p.denominator] == KATS["padding_53_8"] and p == Fraction(53, 56)
    kr = ukernel.UKernel(reg_tile={"i": 4, "j": 4}, smem_tile={"i": 32, "j": 32, "k": 8})
    assert metrics.regs_in_block(kr, hw80()) == KATS["regs_4x4_32x32"] == 2048
    k2 = ukernel.UKernel(reg_tile={"i": 1, "j": 1}, smem_tile={"i": 32, "j": 64, "k": 8})
    assert metrics.space_saturation(k2, inst, hw80()) == KATS["saturation_128x2304_32x64"] is False
    cube = workload.WorkloadInstance(workload.parse_workload(dense_doc(128, 128, 4, 8192)), {"i": 128})
    kc = ukernel.UKernel(reg_tile={"i": 1, "j": 1}, smem_tile={"i": 128, "j": 128, "k": 128})
    assert workload.data_volumes(cube, kc) == KATS["data_volumes_128"]


def test_select_main_axis():
    inst = workload.WorkloadInstance(workload.parse_workload(dense_doc(2304, 768, 4, 8192)), {"i": 53})
    assert combine.select_main_axis(inst) == "j"
    inst = workload.WorkloadInstance(workload.parse_workload(dense_doc(768, 768, 4, 8192)), {"i": 768})
    assert combine.select_main_axis(inst) == "i"


def test_descriptor_roundtrip_and_errors():
    from paper_2407_21418_b200.mktune import errors, hardware

    d = hardware.b200_bf16(tcgen05=True)
    assert hardware.load_hardware_descriptor(hardware.serialize_hardware_descriptor(d)) == d
    doc = hardware.b200_ffma().to_doc()
    assert hardware.canonical_document(doc) == hardware.serialize_hardware_descriptor(hardware.load_hardware_descriptor(doc))
    with pytest.raises(errors.InputError) as e:
        hardware.load_hardware_descriptor({**doc, "num_cores": 0})
    assert e.value.field == "num_cores"
    with pytest.raises(errors.InputError) as e:
        hardware.load_hardware_descriptor({**doc, "bogus": 1})
    assert e.value.field == "bogus"
    with pytest.raises(errors.InputError):
        hardware.load_hardware_descriptor({**doc, "align_elems": 48})


def test_legality_derives_from_the_tcgen05_descriptor():
    """the B200 legality rules come from the descriptor's
    tcgen05 fields, not constants. With mma_n_max = 128 (and 256 TMEM
    columns) the widest column tile is 128: every plan's output tiles are
    whole 128-lane slabs / 128-column MMA tiles or span a short axis, and the
    256-column plans of the sm_100a descriptor disappear. A 64-B swizzle
    makes 32-element reduce tiles legal; invalid values are InputErrors."""
    import dataclasses

    import pytest

    from paper_2407_21418_b200.mktune.errors import InputError
    from paper_2407_21418_b200.mktune.hardware import b200_bf16
    from paper_2407_21418_b200.runtime import Planner, bmm_instance, dense_instance

    base = b200_bf16(tcgen05=True)
    narrow = dataclasses.replace(base, mma_n_max=128, tmem_columns=256)
    shapes = [dense_instance(1216, 2304, 768), dense_instance(4096, 768, 768), dense_instance(160, 3072, 768),
              bmm_instance(384, 100, 100, 64)]

    def out_tiles(hw):
        recs = Planner(hw=hw).plan(shapes)
        res = []
        for inst, r in zip(shapes, recs):
            g = r.program
            ns = g.n_space
            res.append([(int(g.smem[p][ns - 2]), int(g.smem[p][ns - 1])) for p in range(g.n_parts)])
        return res, recs

    wide, _ = out_tiles(base)
    slim, recs = out_tiles(narrow)
    assert any(256 in t for tiles in wide for t in tiles), "the sm_100a descriptor picks 256-column tiles"
    assert all(max(t) <= 256 for tiles in slim for t in tiles)
    for inst, tiles, r in zip(shapes, slim, recs):
        ext = [inst.extents[a] for a in inst.spec.space_axes][-2:]
        for ti, tj in tiles:
            ok = lambda lane, col, El, Ec: (((lane % 128 == 0 and lane <= 256) or (El <= lane <= 128))  # noqa: E731
                                             and (col == 128 or Ec <= col <= 128))
            if r.stage < 4:  # strict rung: the narrowed rule holds in one of the two orientations
                assert ok(ti, tj, ext[0], ext[1]) or ok(tj, ti, ext[1], ext[0]), (inst.extents, ti, tj)
    assert slim != wide
    with pytest.raises(InputError):
        dataclasses.replace(base, mma_n_max=384)
    with pytest.raises(InputError):
        dataclasses.replace(base, tmem_columns=256)  # cannot hold two 256-column accumulators
    with pytest.raises(InputError):
        dataclasses.replace(base, mma_m_atoms=(96,))
    # with a 32-element alignment, a 128-B swizzle still demands 64-element
    # reduce tiles (one bf16 swizzle atom); a 64-B swizzle admits 32
    a32 = dataclasses.replace(base, align_elems=32)
    swz64 = dataclasses.replace(a32, tma_swizzle_bytes=64)
    from paper_2407_21418_b200.mktune.ukernel import enumerate_ukernels

    inst = dense_instance(160, 768, 768)
    ks_default = {int(k) for k in enumerate_ukernels(inst, a32).smem[:, 2]}
    ks_64 = {int(k) for k in enumerate_ukernels(inst, swz64).smem[:, 2]}
    assert all(k % 64 == 0 for k in ks_default) and any(k % 64 for k in ks_64)
