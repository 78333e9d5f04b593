"""C++ planner (via the mktune facade) vs golden fixtures generated from the
reference (tests/golden/make_golden.py): candidate sets bit-exact (tile
order, retained steps, every metric incl. float64 bits), relaxation
provenance, pool size and order, Top-10 incl. SIA float bits."""

import pytest

from _helpers import (CASES, GOLDEN, digest_candidates, digest_pool, facade_hw, facade_instance, facade_params,
                      fhex, plan_key, top_rows)

CASE_IDS = [c["id"] for c in CASES if c["id"] in GOLDEN]


def _case(cid):
    return next(c for c in CASES if c["id"] == cid)


@pytest.fixture(scope="module")
def compiled():
    from paper_2407_21418_b200.mktune.filtering import compile_shape

    out = {}
    for cid in CASE_IDS:
        c = _case(cid)
        inst = facade_instance(c)
        out[cid] = (inst, compile_shape(inst, facade_hw(c), facade_params(c)))
    return out


@pytest.mark.parametrize("cid", CASE_IDS)
def test_compile_shape_bitexact(compiled, cid):
    g = GOLDEN[cid]
    inst, r = compiled[cid]
    assert r.counts == g["counts"]
    assert r.relaxation == g["relaxation"]
    assert r.truncated == g["truncated"]
    assert r.sweep_used.to_doc() == g["sweep_used"]
    assert len(r.candidates) == g["n_final"]
    spec = inst.spec
    space, axes = spec.space_axes, tuple(spec.space_axes) + tuple(spec.reduce_axes)
    keys = [k.tile_key(space, axes) for k in r.candidates]
    assert [[list(a), list(b)] for a, b in keys[:5]] == g["head"]
    bundles = [(float(b.pad), float(b.occ), b.regs_in_block, b.saturated, b.cmr, b.mem_latency_s, b.blocks_needed)
               for b in r.bundles]
    assert digest_candidates(keys, r.retained_steps, bundles) == g["cand_digest"]


@pytest.mark.parametrize("cid", CASE_IDS)
def test_topk_streaming_matches_reference(compiled, cid):
    from paper_2407_21418_b200.mktune.combine import plan_pool_size, select_main_axis
    from paper_2407_21418_b200.mktune.scoring import rank_topk

    g = GOLDEN[cid]
    inst, r = compiled[cid]
    assert select_main_axis(inst) == g["tau"]
    assert plan_pool_size(r.candidates, inst) == g["pool_size"]
    if g["pool_size"] == 0:  # the reference raises EmptyResultError from build_programs
        from paper_2407_21418_b200.mktune.errors import EmptyResultError

        with pytest.raises(EmptyResultError):
            rank_topk(r.candidates, inst, k=10)
        return
    top = rank_topk(r.candidates, inst, k=10)
    assert top_rows(top, inst) == [t["parts"] for t in g["top10"]]
    assert [fhex(p.sia) for p in top] == [t["sia"] for t in g["top10"]]
    for p in top:
        assert p.tau_coverage == inst.extent(p.tau)


@pytest.mark.parametrize("cid", [c for c in CASE_IDS if "pool_digest" in GOLDEN[c] and GOLDEN[c]["pool_size"] <= 120_000])
def test_build_programs_and_rank_programs(compiled, cid):
    from paper_2407_21418_b200.mktune.combine import build_programs
    from paper_2407_21418_b200.mktune.scoring import rank_programs

    g = GOLDEN[cid]
    inst, r = compiled[cid]
    pool = build_programs(r.candidates, inst)
    spec = inst.spec
    space, axes = spec.space_axes, tuple(spec.space_axes) + tuple(spec.reduce_axes)
    assert len(pool) == g["pool_size"]
    assert digest_pool([plan_key([(k.tile_key(space, axes), n) for k, n in p.parts]) for p in pool]) == g["pool_digest"]
    top = rank_programs(pool, k=10)
    assert top_rows(top, inst) == [t["parts"] for t in g["top10"]]
    topn = rank_programs(pool, k=10, normalize=True)
    assert top_rows(topn, inst) == [t["parts"] for t in g["top10_normalized"]]
    assert [fhex(p.sia) for p in topn] == [t["sia"] for t in g["top10_normalized"]]
    # the pure-Python path (a plain list) must agree with the native fast path
    plain = list(pool)
    assert top_rows(rank_programs(plain[:5000], k=5), inst) == top_rows(rank_programs(type(pool)(plain[:5000]), k=5), inst)


@pytest.mark.reference
@pytest.mark.parametrize("M", [3, 17, 100, 333])
def test_live_reference_compile(M):
    """Against the reference itself (build container only)."""
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    import mktune.filtering as rf
    import mktune.hardware as rh
    import mktune.workload as rw
    from cases import dense_doc

    from paper_2407_21418_b200.mktune import filtering, hardware, workload
    from _helpers import DESCRIPTORS

    doc = dense_doc(2304, 768, 2)
    rr = rf.compile_shape(rw.WorkloadInstance(rw.parse_workload(doc), {"i": M}), rh.HardwareDescriptor(**DESCRIPTORS["b200_bf16"]))
    mm = filtering.compile_shape(workload.WorkloadInstance(workload.parse_workload(doc), {"i": M}),
                                 hardware.HardwareDescriptor(**DESCRIPTORS["b200_bf16"]))
    assert rr.counts == mm.counts and rr.relaxation == mm.relaxation
    assert [(k.reg_tile, k.smem_tile, k.compute_eff) for k in rr.candidates] == \
        [(k.reg_tile, k.smem_tile, k.compute_eff) for k in mm.candidates]
