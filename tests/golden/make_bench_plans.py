#!/usr/bin/env python3
"""Pin the plans the headline bench actually executes: run the REFERENCE
(mktune 0.1.0 at /root/reference/pkg/src, read-only) on every shape of the
C1 bench set (bench.py: c1_shapes(24, seed=0), 192 GEMMs) in B200 mode, and
write tests/golden/bench_plans.json.

B200 mode in reference terms:
  * the tcgen05 legality filter (_digest.tcgen05_legal, the Python statement
    of planner.cpp tcgen05_legal) is monkeypatched into the reference's
    enumerate_ukernels (bound into mktune.filtering, filtering.py:44-50,277);
  * rung 0 (stage 0): reference compile_shape, then the Top-1 of
    rank_programs(build_programs(...)) (combine.py:133-194, scoring.py:83-126)
    with tau = select_main_axis (combine.py:58-68);
  * rung 1 (reported stage 4, Dense only): taken when no combination of the
    LEGAL ALIGN SET covers the main axis (so neither the final, filter nor
    cross subsets can: stages 0-3 of rung 0 are all empty, checked here by
    counting the align set's pool with reference primitives); the same final
    set is then ranked with tau forced to the other output axis
    (capi.cpp ftb_plan_batch).
Top-1 comes from make_golden.streaming_topk (reference primitives only;
validated against the real build_programs + rank_programs wherever the pool
fits, make_golden.py). Pools here are small (legality-filtered), so every
rung-0 Top-1 is additionally cross-checked against the materialised
reference pool when it holds <= 400k plans.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_bench_plans.py
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(ROOT))

import make_golden as mg  # noqa: E402  (puts the reference on sys.path)
from mktune.combine import _pair_solutions, _part_signature, build_programs, select_main_axis  # noqa: E402
from mktune.filtering import FilterParams, compile_shape  # noqa: E402
from mktune.hardware import HardwareDescriptor  # noqa: E402
from mktune.scoring import rank_programs  # noqa: E402
from mktune.workload import WorkloadInstance, parse_workload  # noqa: E402

from _digest import DESCRIPTORS, fhex  # noqa: E402


def bench_shapes():
    """The bench's C1 set (shape generator only: seeded numpy, no planning)."""
    from paper_2407_21418_b200.workloads import c1_shapes

    return c1_shapes(n_draws=24, seed=0)


def pool_count(kernels, inst, tau):
    """len(build_programs(kernels, inst)) for an arbitrary tau, from reference
    primitives (combine.py:150-180) without materialising plans."""
    spec = inst.spec
    space, axes = spec.space_axes, tuple(spec.space_axes) + tuple(spec.reduce_axes)
    H = inst.extent(tau)
    uniq = {}
    for kk in kernels:
        uniq.setdefault(kk.tile_key(space, axes), kk)
    n = sum(1 for kk in uniq.values() if H % kk.smem_tile[tau] == 0)
    groups = {}
    for key_t, kk in uniq.items():
        groups.setdefault(_part_signature(kk, tau, space, axes), []).append(kk.smem_tile[tau])
    for ts in groups.values():
        for x in range(len(ts)):
            for y in range(x + 1, len(ts)):
                if ts[x] != ts[y]:
                    n += len(list(_pair_solutions(min(ts[x], ts[y]), max(ts[x], ts[y]), H)))
    return n


def plan_shape(sh):
    from paper_2407_21418_b200.mktune.workload import workload_hash  # noqa: F401  (doc only)

    doc = sh.instance().spec.to_doc()
    binding = dict(sh.instance().bindings)
    hw = HardwareDescriptor(**DESCRIPTORS["b200_bf16"])
    inst = WorkloadInstance(parse_workload(doc), binding)
    mg.legal_patch(True)
    try:
        res = compile_shape(inst, hw, FilterParams.default())
        tau_main = select_main_axis(inst)
        top, n_main, tau = mg.streaming_topk(res.candidates, inst, k=1)
        assert tau == tau_main
        stage = 0
        if n_main == 0:
            space = list(inst.spec.space_axes)
            if len(space) != 2:
                raise RuntimeError(f"{sh}: no tau cover and no rung-1 axis (BMM)")
            # rung 0 stages 1-3 rank subsets of the legal align set: all empty
            align = mg.rfilt.enumerate_ukernels(inst, hw, cap=FilterParams.default().candidate_cap)
            align_k = [align[i] for i in range(len(align))]
            assert pool_count(align_k, inst, tau_main) == 0, f"{sh}: rung 0 would have a plan"
            tau = space[1 - space.index(tau_main)]
            top, n_other, _ = mg.streaming_topk(res.candidates, inst, k=1, tau=tau)
            assert n_other > 0, f"{sh}: rung 1 empty too"
            stage = 4
        elif n_main <= mg.POOL_MATERIALISE_MAX:
            ranked = rank_programs(build_programs(res.candidates, inst), k=1)
            space_ax = inst.spec.space_axes
            axes = tuple(space_ax) + tuple(inst.spec.reduce_axes)
            got = [(kk.tile_key(space_ax, axes), n) for kk, n in ranked[0].parts]
            assert got == list(top[0][0]) and fhex(ranked[0].sia) == fhex(top[0][1]), f"{sh}: oracle disagrees"
        parts, sia = top[0]
        space = list(inst.spec.space_axes)
        return {
            "name": sh.name, "batch": sh.batch, "M": sh.M, "N": sh.N, "K": sh.K,
            "relaxation": res.relaxation, "counts": res.counts, "stage": stage, "tau": space.index(tau),
            "parts": [[list(t[0]), list(t[1]), n] for t, n in parts], "sia": fhex(sia),
        }
    finally:
        mg.legal_patch(False)


def digest(rows) -> str:
    h = hashlib.sha256()
    for r in rows:
        h.update(repr((r["tau"], r["parts"], r["sia"], r["stage"])).encode())
    return h.hexdigest()


def main():
    t0 = time.time()
    rows = []
    for sh in bench_shapes():
        rows.append(plan_shape(sh))
    out = {"workload": "bench.py C1: c1_shapes(n_draws=24, seed=0), B200 legality mode", "n": len(rows),
           "digest": digest(rows), "plans": rows, "generate_s": time.time() - t0}
    (HERE / "bench_plans.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"{len(rows)} plans, stage-4 {sum(r['stage'] == 4 for r in rows)}, {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
