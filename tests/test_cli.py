"""CLI front door (SPEC.md:505-568 cmd_tune / cmd_plan /
cmd_emit_loopnest / cmd_sweep and their examples). CPU only."""

import csv
import io
import json
import re

import pytest

from paper_2407_21418_b200 import cli
from paper_2407_21418_b200.mktune.hardware import b200_bf16, serialize_hardware_descriptor


def run(capsys, *argv):
    rc = cli.main(list(argv))
    out, err = capsys.readouterr()
    return rc, out, err


def test_tune_is_deterministic_and_embeds_provenance(tmp_path, capsys):
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    for p in (a, b):
        rc, _, err = run(capsys, "tune", "--workload", "dense:768:768", "--range", "i=1..6", "--out", str(p))
        assert rc == 0, err
    assert a.read_bytes() == b.read_bytes()  # SPEC: rerun -> byte-identical cache
    doc = json.loads(a.read_text())
    assert len(doc["sections"]) == 6  # one section per binding
    for key in ("tool", "perf_model", "descriptor", "workload_hash", "schema"):
        assert doc[key]
    assert all(s["candidates"] for s in doc["sections"].values())


def test_tune_parallel_matches_serial(tmp_path, capsys):
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    assert run(capsys, "tune", "--workload", "dense:768:768", "--range", "i=1..8", "--out", str(a))[0] == 0
    assert run(capsys, "tune", "--workload", "dense:768:768", "--range", "i=1..8", "--workers", "4",
               "--out", str(b))[0] == 0
    assert a.read_bytes() == b.read_bytes()


def test_missing_hardware_file_exits_2_naming_the_path(capsys):
    rc, _, err = run(capsys, "tune", "--workload", "dense:768:768", "--range", "i=1..2",
                     "--hardware", "/nonexistent/hw.json")
    assert rc == 2
    assert "/nonexistent/hw.json" in err


def test_bad_inputs_exit_2(capsys):
    assert run(capsys, "plan", "--workload", "dense:768:768", "--shape", "q=5")[0] == 2  # not a dynamic axis
    assert run(capsys, "plan", "--workload", "dense:768:768")[0] == 2  # no binding
    assert run(capsys, "plan", "--workload", "dense:768:768", "--shape", "i=5", "--coeffs", "1,2")[0] == 2
    assert run(capsys, "sweep", "--workload", "dense:768:768", "--range", "i=5..1")[0] == 2
    assert run(capsys, "emit-loopnest", "--plan", "/nonexistent/plan.json")[0] == 2


def test_degenerate_descriptor_exit_code_and_sweep_rows(tmp_path, capsys):
    d = json.loads(serialize_hardware_descriptor(b200_bf16(False)))
    d["smem_per_core_bytes"], d["name"] = 64, "tiny"
    hw = tmp_path / "tiny.json"
    hw.write_text(json.dumps(d))
    rc, _, err = run(capsys, "plan", "--workload", "dense:768:768", "--shape", "i=8", "--hardware", str(hw))
    assert rc == 2 and "CapacityError" in err
    # sweep: per-shape errors become status rows, the run continues (SPEC cmd_sweep)
    rc, out, _ = run(capsys, "sweep", "--workload", "dense:768:768", "--range", "i=1..3", "--hardware", str(hw))
    rows = list(csv.DictReader(io.StringIO(out)))
    assert rc == 0 and len(rows) == 3 and {r["status"] for r in rows} == {"CapacityError"}


def test_plan_topk_sorted_and_cache_round_trip(tmp_path, capsys):
    cache, p1, p2 = tmp_path / "c.json", tmp_path / "p1.json", tmp_path / "p2.json"
    assert run(capsys, "tune", "--workload", "dense:768:768", "--range", "i=50..55", "--out", str(cache))[0] == 0
    assert run(capsys, "plan", "--workload", "dense:768:768", "--shape", "i=53", "--topk", "5",
               "--out", str(p1))[0] == 0
    assert run(capsys, "plan", "--workload", "dense:768:768", "--shape", "i=53", "--topk", "5",
               "--cache", str(cache), "--out", str(p2))[0] == 0
    d1, d2 = json.loads(p1.read_text()), json.loads(p2.read_text())
    s1, s2 = d1["shapes"][0], d2["shapes"][0]
    assert s1["source"] == "compiled" and s2["source"] == "cache"
    assert [p["parts"] for p in s1["plans"]] == [p["parts"] for p in s2["plans"]]
    scores = [p["sia"] for p in s1["plans"]]
    assert scores == sorted(scores, reverse=True)  # Top-K descending by score
    for p in s1["plans"]:  # coverage: the tau parts tile the extent exactly
        tau = p["tau"]
        ti = d1["axes"]["space"].index(tau)
        assert sum(q["count"] * q["smem"][ti] for q in p["parts"]) == s1["extents"][tau]


def test_plan_with_wrong_cache_exits_2(tmp_path, capsys):
    cache = tmp_path / "c.json"
    assert run(capsys, "tune", "--workload", "dense:768:768", "--range", "i=1..2", "--out", str(cache))[0] == 0
    assert run(capsys, "plan", "--workload", "dense:2304:768", "--shape", "i=1", "--cache", str(cache))[0] == 2


@pytest.mark.parametrize("workload,shape", [("dense:768:768", ["i=53"]), ("dense:32:64", ["i=53"]),
                                            ("bmm:12", ["i=38", "j=38", "k=64"])])
def test_emit_loopnest_bounds_reconstruct_covered_extents(tmp_path, capsys, workload, shape):
    plan = tmp_path / "p.json"
    args = ["plan", "--workload", workload, "--topk", "10", "--out", str(plan)]
    for s in shape:
        args += ["--shape", s]
    assert run(capsys, *args)[0] == 0
    doc = json.loads(plan.read_text())
    sh = doc["shapes"][0]
    for idx in range(len(sh["plans"])):
        rc, text, _ = run(capsys, "emit-loopnest", "--plan", str(plan), "--index", str(idx))
        assert rc == 0
        p = sh["plans"][idx]
        nests = text.split("// part ")[1:]
        assert len(nests) == len(p["parts"])  # one nest per part
        tau_cover = 0
        for nest, part in zip(nests, p["parts"]):
            blocks = dict((a, (int(lo), int(hi), int(st))) for a, lo, hi, st in
                          re.findall(r"for (\w+)\.0 in range\((\d+), (\d+), (\d+)\):", nest))
            for a, (lo, hi, st) in blocks.items():
                assert (hi - lo) % st == 0
                if a == p["tau"]:
                    tau_cover += hi - lo
                else:
                    assert hi >= sh["extents"][a] > hi - st  # covered extent = ceil(E/t)*t
            # register tiles innermost, then thread tiles, then block tiles (i.2 inside i.1 inside i.0)
            for a in doc["axes"]["space"]:
                assert nest.index(f"for {a}.0") < nest.index(f"for {a}.1") < nest.index(f"for {a}.2")
        assert tau_cover == sh["extents"][p["tau"]]


V100_LIKE = {"name": "v100-like", "num_cores": 80, "regs_per_core": 65536, "smem_per_core_bytes": 98304,
             "global_bw_bytes_per_s": 900000000000, "shared_bw_bytes_per_s": 15700000000000,
             "peak_flops": 15700000000000, "default_active_blocks": 2, "active_blocks_per_core": 2,
             "align_elems": 8}  # SURVEY Appendix B's comparison descriptor


def test_two_part_plan_gets_two_nests_with_offset(tmp_path, capsys):
    """A dynamic tau (N=16 < M=53, so tau=i) covered by two tile sizes emits
    two nests, the second at a tau offset (SPEC cmd_emit_loopnest example)."""
    hw, plan = tmp_path / "v100.json", tmp_path / "p.json"
    hw.write_text(json.dumps(V100_LIKE))
    assert run(capsys, "plan", "--workload", "dense:16:256:4", "--shape", "i=53", "--topk", "20",
               "--hardware", str(hw), "--out", str(plan))[0] == 0
    sh = json.loads(plan.read_text())["shapes"][0]
    assert sh["tau"] == "i"
    two = [i for i, p in enumerate(sh["plans"]) if len(p["parts"]) == 2]
    assert two
    rc, text, _ = run(capsys, "emit-loopnest", "--plan", str(plan), "--index", str(two[0]))
    assert rc == 0
    offs = re.findall(r"at \w+ offset (\d+)", text)
    assert len(offs) == 2 and offs[0] == "0" and int(offs[1]) > 0
    blocks = re.findall(r"for i\.0 in range\((\d+), (\d+), (\d+)\):", text)
    assert sum(int(hi) - int(lo) for lo, hi, _ in blocks) == 53


def test_empty_result_exits_1(tmp_path, capsys):
    hw = tmp_path / "v100.json"
    hw.write_text(json.dumps(V100_LIKE))
    rc, _, err = run(capsys, "plan", "--workload", "dense:32:768:4", "--shape", "i=53", "--hardware", str(hw))
    assert rc == 1 and "EmptyResultError" in err


def test_sweep_rows_and_padding_definition(capsys):
    rc, out, err = run(capsys, "sweep", "--workload", "dense:768:768", "--range", "i=1..16")
    assert rc == 0, err
    rows = list(csv.DictReader(io.StringIO(out)))
    assert len(rows) == 16 and all(r["status"] == "ok" for r in rows)
    for r in rows:
        assert 0.0 <= float(r["padding_fraction"]) < 1.0
        assert float(r["est_total_s"]) > 0


def test_env_overrides(monkeypatch, capsys):
    monkeypatch.setenv("FTB_CLI_WORKLOAD", "dense:768:768")
    monkeypatch.setenv("FTB_CLI_RANGE", "i=1..3")
    rc, out, _ = run(capsys, "sweep")
    assert rc == 0 and len(out.strip().splitlines()) == 4


def test_plan_report_is_byte_identical_and_timings_go_elsewhere(tmp_path, capsys):
    """SPEC invariant "All commands are deterministic": the plan report holds
    no wall-clock; --timings writes the combine + rank times to its own file."""
    a, b, t = tmp_path / "a.json", tmp_path / "b.json", tmp_path / "t.json"
    for p in (a, b):
        rc, _, err = run(capsys, "plan", "--workload", "dense:768:768", "--range", "i=50..53", "--topk", "3",
                         "--out", str(p), "--timings", str(t))
        assert rc == 0, err
    assert a.read_bytes() == b.read_bytes()
    assert "timing" not in a.read_text()
    tim = json.loads(t.read_text())
    assert tim["kind"] == "plan-timings" and len(tim["shapes"]) == 4
    assert all(s["combine_rank_s"] >= 0 for s in tim["shapes"])


def test_env_overrides_flags_that_have_defaults(tmp_path, capsys, monkeypatch):
    """FTB_CLI_* applies to --topk / --emit too (defaults resolve after the
    environment); a flag on the command line still wins."""
    out = tmp_path / "p.json"
    monkeypatch.setenv("FTB_CLI_TOPK", "2")
    assert run(capsys, "plan", "--workload", "dense:768:768", "--shape", "i=53", "--out", str(out))[0] == 0
    assert len(json.loads(out.read_text())["shapes"][0]["plans"]) == 2
    assert run(capsys, "plan", "--workload", "dense:768:768", "--shape", "i=53", "--topk", "4",
               "--out", str(out))[0] == 0
    assert len(json.loads(out.read_text())["shapes"][0]["plans"]) == 4
    monkeypatch.setenv("FTB_CLI_EMIT", "csv")
    assert run(capsys, "plan", "--workload", "dense:768:768", "--shape", "i=53", "--out", str(out))[0] == 0
    rows = list(csv.DictReader(io.StringIO(out.read_text())))
    assert [int(r["rank"]) for r in rows] == [0, 1]
    assert all(r["binding"] == "i=53" for r in rows)
