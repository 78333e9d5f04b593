#!/usr/bin/env python3
"""Generate tests/golden/*.json by running the REFERENCE (mktune 0.1.0 at
/root/reference/pkg/src, read-only) in the build container.

The reference cannot travel to the GPU box, so its outputs are committed as
fixtures. For pools too large to materialise (millions of ProgramPlan
objects) the Top-10 is computed by a streaming oracle assembled only from
reference primitives (select_main_axis, _part_signature, _pair_solutions,
the cached part metrics and the rank key of scoring.py:120-123), as
SURVEY.md §4 item 1 prescribes; it is validated against the real
build_programs + rank_programs on every case whose pool fits.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
"""

from __future__ import annotations

import heapq
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

import mktune.filtering as rfilt  # noqa: E402
from mktune.combine import _pair_solutions, _part_signature, build_programs, select_main_axis  # noqa: E402
from mktune.filtering import FilterParams, compile_shape  # noqa: E402
from mktune.hardware import HardwareDescriptor  # noqa: E402
from mktune.scoring import SiaCoeffs, rank_programs  # noqa: E402
from mktune.ukernel import enumerate_ukernels  # noqa: E402
from mktune.workload import WorkloadInstance, parse_workload  # noqa: E402

from _digest import DESCRIPTORS, digest_candidates, digest_pool, fhex, plan_key, tcgen05_legal  # noqa: E402
from cases import CASES  # noqa: E402

POOL_MATERIALISE_MAX = 400_000


def streaming_topk(kernels, inst, k=10, coeffs=None, tau=None):
    """Top-k of rank_programs(build_programs(kernels, inst)) from reference
    primitives; ``tau`` overrides select_main_axis (B200 fallback rung 1)."""
    coeffs = coeffs or SiaCoeffs()
    spec = inst.spec
    space, axes = spec.space_axes, tuple(spec.space_axes) + tuple(spec.reduce_axes)
    tau = select_main_axis(inst) if tau is None else tau
    H = inst.extent(tau)
    uniq = {}
    for kk in kernels:
        uniq.setdefault(kk.tile_key(space, axes), kk)

    def part(kk):
        return coeffs.c0 * kk.compute_eff + coeffs.c1 * kk.padding_threshold + coeffs.c2 * kk.usage_eff

    heap = []  # max-heap on the rank key via negation wrapper

    class Neg:
        __slots__ = ("key", "item")

        def __init__(self, key, item):
            self.key, self.item = key, item

        def __lt__(self, other):
            return self.key > other.key

    def offer(key, item):
        if len(heap) < k:
            heapq.heappush(heap, Neg(key, item))
            return True
        if key < heap[0].key:
            heapq.heapreplace(heap, Neg(key, item))
            return True
        return False

    n_plans = 0
    for key_t, kk in uniq.items():
        t = kk.smem_tile[tau]
        if H % t == 0:
            n_plans += 1
            s = sum([part(kk)]) / 1
            offer((-s, 1, -kk.padding_threshold, ((key_t, H // t),)), (((key_t, H // t),), s))
    groups = {}
    for key_t, kk in uniq.items():
        groups.setdefault(_part_signature(kk, tau, space, axes), []).append((key_t, kk))
    for members in groups.values():
        members.sort(key=lambda x: x[0])
        for x in range(len(members)):
            k1t, k1 = members[x]
            a = k1.smem_tile[tau]
            for y in range(x + 1, len(members)):
                k2t, k2 = members[y]
                b = k2.smem_tile[tau]
                if a == b:
                    continue
                (lt, lk), (ht, hk) = ((k1t, k1), (k2t, k2)) if a < b else ((k2t, k2), (k1t, k1))
                sols = list(_pair_solutions(min(a, b), max(a, b), H))
                n_plans += len(sols)
                if not sols:
                    continue
                s = sum([part(lk), part(hk)]) / 2
                mp = sum([lk.padding_threshold, hk.padding_threshold]) / 2
                for n1, n2 in reversed(sols):  # ascending n1 = ascending tile order
                    key = (-s, 2, -mp, ((lt, n1), (ht, n2)))
                    if not offer(key, (((lt, n1), (ht, n2)), s)):
                        break
    out = sorted(heap, key=lambda w: w.key)
    return [w.item for w in out], n_plans, tau


def legal_patch(enabled):
    orig = enumerate_ukernels

    def patched(instance, hw, cap=None, major_axis=None):
        cs = orig(instance, hw, cap=cap, major_axis=major_axis)
        if not enabled:
            return cs
        import numpy as np

        space = instance.spec.space_axes
        axes = cs.axis_names
        ext = instance.extents
        keep = [i for i in range(len(cs)) if tcgen05_legal(space, ext, dict(zip(axes, map(int, cs.smem[i]))))]
        return cs.subset(np.asarray(keep, dtype=np.int64))

    rfilt.enumerate_ukernels = patched


def run_case(case):
    hw = HardwareDescriptor(**DESCRIPTORS[case["hw"]])
    spec = parse_workload(case["doc"])
    inst = WorkloadInstance(spec, dict(case["binding"]))
    legal_patch(case["legal"])
    params = FilterParams.default()
    params.candidate_cap = case["cap"]
    t0 = time.time()
    res = compile_shape(inst, hw, params)
    t_compile = time.time() - t0
    space, axes = spec.space_axes, tuple(spec.space_axes) + tuple(spec.reduce_axes)
    keys = [kk.tile_key(space, axes) for kk in res.candidates]
    bundles = [(float(b.pad), float(b.occ), b.regs_in_block, b.saturated, b.cmr, b.mem_latency_s, b.blocks_needed)
               for b in res.bundles]
    out = {
        "id": case["id"],
        "counts": res.counts, "relaxation": res.relaxation, "truncated": res.truncated,
        "sweep_used": res.sweep_used.to_doc(), "n_final": len(res.candidates),
        "retained_head": list(res.retained_steps[:20]),
        "head": [[list(r), list(s)] for r, s in keys[:5]],
        "cand_digest": digest_candidates(keys, res.retained_steps, bundles),
        "compile_s_reference": t_compile,
    }
    top, n_plans, tau = streaming_topk(res.candidates, inst, k=10)
    out["tau"] = tau
    out["pool_size"] = n_plans
    out["top10"] = [{"parts": [[list(t[0]), list(t[1]), n] for t, n in parts], "sia": fhex(s)} for parts, s in top]
    if 0 < n_plans <= POOL_MATERIALISE_MAX:
        t0 = time.time()
        pool = build_programs(res.candidates, inst)
        ranked = rank_programs(pool, k=10)
        ranked_n = rank_programs(pool, k=10, normalize=True)
        out["build_rank_s_reference"] = time.time() - t0
        pk = [plan_key([(kk.tile_key(space, axes), n) for kk, n in p.parts]) for p in pool]
        out["pool_digest"] = digest_pool(pk)
        ref_top = [[[list(kk.tile_key(space, axes)[0]), list(kk.tile_key(space, axes)[1]), n] for kk, n in p.parts]
                   for p in ranked]
        assert ref_top == [t["parts"] for t in out["top10"]], f"streaming oracle disagrees on {case['id']}"
        assert [fhex(p.sia) for p in ranked] == [t["sia"] for t in out["top10"]]
        out["top10_normalized"] = [{"parts": [[list(kk.tile_key(space, axes)[0]), list(kk.tile_key(space, axes)[1]), n]
                                              for kk, n in p.parts], "sia": fhex(p.sia)} for p in ranked_n]
        out["streaming_validated"] = True
    legal_patch(False)
    return out


def kats():
    """Known answers from SPEC.md examples, computed by the reference."""
    from mktune.combine import combin_search
    from mktune.metrics import occupancy_metric, padding_metric, regs_in_block, space_saturation
    from mktune.oracles import brute_force_combinations, random_combination_case
    from mktune.ukernel import UKernel, reg_tile_candidates
    from mktune.workload import data_volumes, flops

    d = {}
    d["combin_53_7_8"] = sorted(combin_search([7, 8], 53))
    d["reg_tile_53_8"] = reg_tile_candidates(53, 8)
    d["random_cases"] = []
    for seed in range(0, 1000, 37):
        c = random_combination_case(seed)
        d["random_cases"].append({"seed": seed, "tiles": list(c.tiles), "extent": c.extent,
                                  "expected": sorted(brute_force_combinations(c.tiles, c.extent))})
    hw80 = HardwareDescriptor(**{**DESCRIPTORS["v100_like"]})
    spec = parse_workload({**__import__("cases").dense_doc(2304, 768, 4, 8192)})
    occ = {}
    # occupancy on 80 cores for n = 80, 81, 160 blocks
    occ_spec = parse_workload(__import__("cases").dense_doc(1, 64, 4, 8192))
    for n in (80, 81, 160):
        inst = WorkloadInstance(occ_spec, {"i": n})
        k = UKernel(reg_tile={"i": 1, "j": 1}, smem_tile={"i": 1, "j": 8, "k": 8})
        f = occupancy_metric(k, inst, hw80)
        occ[str(n)] = [f.numerator, f.denominator]
    d["occupancy_80"] = occ
    inst = WorkloadInstance(spec, {"i": 128})
    d["flops_128_2304_768"] = flops(inst)
    inst53 = WorkloadInstance(parse_workload(__import__("cases").dense_doc(768, 768, 4, 8192)), {"i": 53})
    k = UKernel(reg_tile={"i": 1, "j": 8}, smem_tile={"i": 8, "j": 64, "k": 64})
    p = padding_metric(k, inst53)
    d["padding_53_8"] = [p.numerator, p.denominator]
    d["regs_4x4_32x32"] = regs_in_block(UKernel(reg_tile={"i": 4, "j": 4}, smem_tile={"i": 32, "j": 32, "k": 8}), hw80)
    k2 = UKernel(reg_tile={"i": 1, "j": 1}, smem_tile={"i": 32, "j": 64, "k": 8})
    d["saturation_128x2304_32x64"] = space_saturation(k2, inst, hw80)
    cube = parse_workload(__import__("cases").dense_doc(128, 128, 4, 8192))
    kc = UKernel(reg_tile={"i": 1, "j": 1}, smem_tile={"i": 128, "j": 128, "k": 128})
    d["data_volumes_128"] = data_volumes(WorkloadInstance(cube, {"i": 128}), kc)
    return d


def main():
    """make_golden.py [ids...]            run cases into planner_cases.json
    make_golden.py --part DIR ids...     cases into DIR/<id>.json (for parallel runs)
    make_golden.py --merge DIR           merge DIR/*.json into planner_cases.json"""
    out_p = HERE / "planner_cases.json"
    existing = json.loads(out_p.read_text()) if out_p.exists() else {}
    if sys.argv[1:2] == ["--part"]:
        part = Path(sys.argv[2])
        part.mkdir(parents=True, exist_ok=True)
        for case in CASES:
            if case["id"] in sys.argv[3:]:
                t0 = time.time()
                res = run_case(case)
                (part / f"{case['id']}.json").write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")
                print(f"{case['id']}: {time.time() - t0:.1f}s pool={res['pool_size']}", flush=True)
        return
    if sys.argv[1:2] == ["--merge"]:
        for p in sorted(Path(sys.argv[2]).glob("*.json")):
            existing[p.stem] = json.loads(p.read_text())
        out_p.write_text(json.dumps(existing, indent=1, sort_keys=True) + "\n")
        return
    only = set(sys.argv[1:])
    for case in CASES:
        if only and case["id"] not in only:
            continue
        t0 = time.time()
        existing[case["id"]] = run_case(case)
        print(f"{case['id']}: {time.time() - t0:.1f}s pool={existing[case['id']]['pool_size']}", flush=True)
        out_p.write_text(json.dumps(existing, indent=1, sort_keys=True) + "\n")
    (HERE / "kats.json").write_text(json.dumps(kats(), indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
