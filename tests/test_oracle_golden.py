"""Pin the oracle port (oracle/planner_port.py) against the reference's
golden fixtures before trusting it as the checker."""

import numpy as np
import pytest

from _helpers import CASES, DESCRIPTORS, GOLDEN, digest_candidates, fhex, tcgen05_legal
from oracle import planner_port as P

IDS = [c["id"] for c in CASES if c["id"] in GOLDEN and not c["big"]]


def _spec(case):
    doc = case["doc"]
    eb = doc["elem_bytes"]
    return P.dense_spec(eb) if len(doc["axes"]) == 3 else P.bmm_spec(eb)


def _ext(case):
    e = {}
    for a in case["doc"]["axes"]:
        e[a["name"]] = case["binding"][a["name"]] if "range" in a else a["extent"]
    return e


@pytest.mark.parametrize("cid", IDS)
def test_port_matches_reference(cid):
    case = next(c for c in CASES if c["id"] == cid)
    g = GOLDEN[cid]
    spec, ext = _spec(case), _ext(case)
    legal = (lambda sm: tcgen05_legal(spec.space, ext, sm)) if case["legal"] else None
    so = P.compile_shape(spec, ext, DESCRIPTORS[case["hw"]], cap=case["cap"], legal=legal)
    assert so.counts == g["counts"]
    assert so.relaxation == g["relaxation"]
    assert so.truncated == g["truncated"]
    keys = [(tuple(map(int, r)), tuple(map(int, s))) for r, s in zip(so.reg, so.smem)]
    c = so.cols
    bundles = [(float(c["pad_num"][i] / c["pad_den"][i]), float(c["blocks"][i] / c["occ_den"][i]),
                int(c["regs_in_block"][i]), bool(c["saturated"][i]), float(c["cmr"][i]), float(c["kmem"][i]),
                int(c["blocks"][i])) for i in range(len(keys))]
    assert digest_candidates(keys, [int(v) for v in so.retained], bundles) == g["cand_digest"]
    dyn = {a["name"] for a in case["doc"]["axes"] if "range" in a}
    assert P.main_axis(spec, ext, dyn) == g["tau"]
    if g["pool_size"] <= 120_000:
        pool = P.build_pool(spec, so, g["tau"])
        assert len(pool) == g["pool_size"]
        top = P.rank(spec, so, pool, 10)
        assert [fhex(s) for _, s, _ in top] == [t["sia"] for t in g["top10"]]
        assert [[[list(k[0]), list(k[1]), n] for k, n in t] for _, _, t in top] == [t["parts"] for t in g["top10"]]


def test_pair_counts_vs_bruteforce():
    rng = np.random.default_rng(0)
    for _ in range(300):
        a, b = sorted(rng.choice(np.arange(1, 65), 2, replace=False))
        H = int(rng.integers(1, 513))
        brute = [(n1, (H - n1 * a) // b) for n1 in range(1, H) if H - n1 * a >= b and (H - n1 * a) % b == 0]
        assert sorted(P.pair_counts(int(a), int(b), H)) == sorted(brute)
