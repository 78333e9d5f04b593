"""Shared test helpers: build facade / oracle objects from golden cases."""

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))

from _digest import DESCRIPTORS, digest_candidates, digest_pool, fhex, plan_key, tcgen05_legal  # noqa: E402,F401
from cases import CASES  # noqa: E402,F401

GOLDEN = json.loads((HERE / "golden" / "planner_cases.json").read_text()) if (HERE / "golden" / "planner_cases.json").exists() else {}
KATS = json.loads((HERE / "golden" / "kats.json").read_text()) if (HERE / "golden" / "kats.json").exists() else {}


def facade_hw(case):
    from paper_2407_21418_b200.mktune.hardware import EXT_FIELDS, HardwareDescriptor

    d = dict(DESCRIPTORS[case["hw"]])
    if case["legal"]:
        d.update(EXT_FIELDS)
    return HardwareDescriptor(**d)


def facade_instance(case):
    from paper_2407_21418_b200.mktune.workload import WorkloadInstance, parse_workload

    return WorkloadInstance(parse_workload(case["doc"]), dict(case["binding"]))


def facade_params(case):
    from paper_2407_21418_b200.mktune.filtering import FilterParams

    p = FilterParams.default()
    p.candidate_cap = case["cap"]
    return p


def top_rows(plans, inst):
    spec = inst.spec
    space, axes = spec.space_axes, tuple(spec.space_axes) + tuple(spec.reduce_axes)
    return [[[list(k.tile_key(space, axes)[0]), list(k.tile_key(space, axes)[1]), n] for k, n in p.parts] for p in plans]
