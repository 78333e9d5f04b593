"""Batch front door (the CLI module of the reference's
SPEC.md:505-568, whose console script `mktune.cli` is declared but absent,
pyproject.toml:25-26).

    python -m paper_2407_21418_b200.cli tune  --workload W.json --range i=1..128 --out cache.json
    python -m paper_2407_21418_b200.cli plan  --workload W.json --shape i=53 [--cache cache.json] --out plan.json
    python -m paper_2407_21418_b200.cli emit-loopnest --plan plan.json [--index 0]
    python -m paper_2407_21418_b200.cli sweep --workload W.json --range i=1..128 --out sweep.csv

``--workload`` takes a workload JSON file (SPEC's document format) or a
preset ``dense:N:K[:elem_bytes]`` / ``bmm:B[:elem_bytes]`` (i, j, k dynamic
for BMM: bind them with --shape/--range). ``--hardware`` takes a descriptor
JSON file or a preset: ``b200-bf16`` (tcgen05 legality, the default),
``b200-bf16-parity`` (the reference's 9 fields only), ``b200-ffma``.
Every flag has an environment override ``FTB_CLI_<FLAG>`` (upper case,
dashes -> underscores), used when the flag is absent.

Exit codes (errors.py:3-4): 0 success, 1 empty result,
2 input error, 3 internal invariant violation. All outputs are
deterministic for identical inputs (sorted keys, no timestamps; wall-clock
fields are confined to the plan report's ``timing`` object) and embed the
tool version, perf-model version, descriptor name and workload hash.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import sys
import time
from pathlib import Path

from . import __version__
from .mktune import errors as E
from .mktune.combine import select_main_axis
from .mktune.filtering import FilterParams, SweepParams, compile_shape, compile_stage
from .mktune.hardware import b200_bf16, b200_ffma, load_hardware_file
from .mktune.scoring import SiaCoeffs, rank_topk, score_decomposition
from .mktune.timemodel import PERF_MODEL_VERSION, estimate_time
from .mktune.ukernel import UKernel
from .mktune.workload import (WorkloadInstance, bmm_spec, dense_spec, load_workload_file, workload_hash)

SCHEMA = 1  # cache / plan / CSV schema integer (bumped on breaking changes)


# ---------------------------------------------------------------- inputs

def _hardware(arg: str | None):
    name = arg or "b200-bf16"
    presets = {"b200-bf16": lambda: b200_bf16(True), "b200-bf16-parity": lambda: b200_bf16(False),
               "b200-ffma": b200_ffma}
    if name in presets:
        return presets[name]()
    p = Path(name)
    if not p.exists():
        raise E.InputError(f"hardware file not found: {p}", field="hardware")
    return load_hardware_file(p)


def _workload(arg: str | None):
    if not arg:
        raise E.InputError("--workload is required (a JSON file or dense:N:K / bmm:B)", field="workload")
    if arg.startswith("dense:"):
        f = arg.split(":")[1:]
        if len(f) not in (2, 3):
            raise E.InputError(f"bad dense preset '{arg}' (dense:N:K[:elem_bytes])", field="workload")
        n, k = int(f[0]), int(f[1])
        return dense_spec(n, k, elem_bytes=int(f[2]) if len(f) == 3 else 2)
    if arg.startswith("bmm:"):
        f = arg.split(":")[1:]
        if len(f) not in (1, 2):
            raise E.InputError(f"bad bmm preset '{arg}' (bmm:B[:elem_bytes])", field="workload")
        return bmm_spec(int(f[0]), i=(1, 512), j=(1, 512), k=(1, 512), elem_bytes=int(f[1]) if len(f) == 2 else 2)
    return load_workload_file(arg)


def _kv(item: str, flag: str) -> tuple[str, str]:
    if "=" not in item:
        raise E.InputError(f"{flag} expects NAME=VALUE, got '{item}'", field=flag.lstrip("-"))
    k, v = item.split("=", 1)
    return k.strip(), v.strip()


def _bindings(spec, shapes: list[str], ranges: list[str]) -> list[dict]:
    """Cartesian product of --range spans and fixed --shape values, in
    binding order (first dynamic axis outermost), validated against the spec."""
    fixed, spans = {}, {}
    for s in shapes or []:
        k, v = _kv(s, "--shape")
        fixed[k] = int(v)
    for r in ranges or []:
        k, v = _kv(r, "--range")
        if ".." not in v:
            raise E.InputError(f"--range expects NAME=LO..HI, got '{r}'", field="range")
        lo, hi = (int(x) for x in v.split("..", 1))
        if hi < lo:
            raise E.InputError(f"empty range '{r}'", field="range")
        spans[k] = range(lo, hi + 1)
    dyn = list(spec.dynamic_axes)
    for name in list(fixed) + list(spans):
        if name not in dyn:
            raise E.InputError(f"'{name}' is not a dynamic axis of {spec.name} (dynamic: {dyn})", field=name)
    missing = [a for a in dyn if a not in fixed and a not in spans]
    if missing:
        raise E.InputError(f"no value for dynamic axis '{missing[0]}' (use --shape or --range)", field=missing[0])
    out = [{}]
    for a in dyn:
        vals = [fixed[a]] if a in fixed else list(spans[a])
        out = [dict(b, **{a: v}) for b in out for v in vals]
    for b in out:  # range checks (WorkloadInstance validates too; fail before any work)
        WorkloadInstance(spec=spec, bindings=b)
    return out


def _params(args) -> FilterParams:
    p = FilterParams(sweep=SweepParams())
    if args.psi is not None:
        p.psi = float(args.psi)
    return p


def _coeffs(arg: str | None) -> SiaCoeffs:
    if not arg:
        return SiaCoeffs()
    try:
        c = [float(x) for x in arg.split(",")]
    except ValueError as exc:
        raise E.InputError(f"--coeffs expects c0,c1,c2, got '{arg}'", field="coeffs") from exc
    if len(c) != 3:
        raise E.InputError(f"--coeffs expects three values, got '{arg}'", field="coeffs")
    return SiaCoeffs(*c)


def _provenance(spec, hw) -> dict:
    return {"schema": SCHEMA, "tool": f"paper_2407_21418_b200 {__version__}", "perf_model": PERF_MODEL_VERSION,
            "descriptor": hw.name, "workload": spec.name, "workload_hash": workload_hash(spec)}


def _binding_key(b: dict) -> str:
    return ",".join(f"{k}={v}" for k, v in sorted(b.items()))


def _write(text: str, out: str | None) -> None:
    if out and out != "-":
        Path(out).write_text(text)
    else:
        sys.stdout.write(text)


# ---------------------------------------------------------------- plan documents

def _kernel_doc(k: UKernel, spec) -> dict:
    return {"reg": [int(k.reg_tile[a]) for a in spec.space_axes],
            "smem": [int(k.smem_tile[a]) for a in list(spec.space_axes) + list(spec.reduce_axes)]}


def _plan_doc(plan, inst, hw, coeffs) -> dict:
    spec = inst.spec
    parts = []
    for (k, n), dec in zip(plan.parts, score_decomposition(plan, coeffs)):
        parts.append(dict(_kernel_doc(k, spec), count=int(n), pad=k.padding_threshold, occ=k.usage_eff,
                          cmr=k.compute_eff, score_terms=dec))
    est = estimate_time(plan, inst, hw)
    tau = plan.tau
    covered, true = 1, 1
    for s in spec.space_axes:
        e = inst.extent(s)
        true *= e
        if s == tau:
            covered *= e
        else:
            t = plan.parts[0][0].smem_tile[s]
            covered *= -(-e // t) * t
    return {"tau": tau, "sia": plan.sia, "parts": parts, "estimate": est.to_doc(),
            "padding_fraction": (covered - true) / covered}


def _candidates_from_cache(cache: dict, spec, hw, binding: dict):
    if cache.get("workload_hash") != workload_hash(spec) or cache.get("descriptor") != hw.name:
        raise E.InputError("cache was made for a different workload or descriptor", field="cache")
    sec = cache.get("sections", {}).get(_binding_key(binding))
    if sec is None:
        return None
    space, axes = list(spec.space_axes), list(spec.space_axes) + list(spec.reduce_axes)
    return [UKernel(reg_tile=dict(zip(space, c["reg"])), smem_tile=dict(zip(axes, c["smem"])),
                    padding_threshold=c["pad"], usage_eff=c["occ"], compute_eff=c["cmr"])
            for c in sec["candidates"]]


# ---------------------------------------------------------------- commands

def cmd_tune(args) -> int:
    """Compile stage over the bindings -> candidate cache (SPEC cmd_tune)."""
    hw, spec = _hardware(args.hardware), _workload(args.workload)
    bindings = _bindings(spec, args.shape, args.range)
    res = compile_stage(spec, hw, _params(args), bindings=bindings, workers=args.workers)
    sections = {}
    for sec in res.sections:
        sections[_binding_key(sec.binding)] = {
            "binding": sec.binding, "counts": sec.counts, "relaxation": sec.relaxation, "truncated": sec.truncated,
            "candidates": [dict(_kernel_doc(k, spec), pad=k.padding_threshold, occ=k.usage_eff, cmr=k.compute_eff)
                           for k in sec.candidates],
        }
    doc = dict(_provenance(spec, hw), kind="candidate-cache", psi=_params(args).psi, sections=sections)
    _write(json.dumps(doc, sort_keys=True, indent=1) + "\n", args.out)
    return 0


def cmd_plan(args) -> int:
    """Runtime stage: combine + SIA Top-K per binding (SPEC cmd_plan)."""
    hw, spec = _hardware(args.hardware), _workload(args.workload)
    coeffs = _coeffs(args.coeffs)
    cache = json.loads(Path(args.cache).read_text()) if args.cache else None
    if args.cache and cache.get("kind") != "candidate-cache":
        raise E.InputError(f"{args.cache} is not a candidate cache", field="cache")
    shapes, timings = [], []
    for b in _bindings(spec, args.shape, args.range):
        inst = WorkloadInstance(spec=spec, bindings=b)
        cands = _candidates_from_cache(cache, spec, hw, b) if cache else None
        source = "cache" if cands is not None else "compiled"
        t0 = time.perf_counter()
        if cands is None:
            cands = compile_shape(inst, hw, _params(args)).candidates
        t1 = time.perf_counter()
        top = rank_topk(cands, inst, coeffs=coeffs, k=args.topk)
        t2 = time.perf_counter()
        shapes.append({"binding": b, "extents": inst.extents, "candidates": len(cands), "source": source,
                       "tau": select_main_axis(inst), "plans": [_plan_doc(p, inst, hw, coeffs) for p in top]})
        timings.append({"binding": b, "compile_s": t1 - t0, "combine_rank_s": t2 - t1})
    doc = dict(_provenance(spec, hw), kind="plan-report", coeffs=coeffs.to_doc(), topk=args.topk,
               axes={"space": list(spec.space_axes), "reduce": list(spec.reduce_axes)},
               inputs=[[a.tensor, list(a.axes)] for a in spec.input_accesses],
               output=[spec.output_access.tensor, list(spec.output_access.axes)], shapes=shapes)
    # The plan report is deterministic (SPEC "All commands are deterministic");
    # the wall-clock of combine + rank (SPEC cmd_plan: "recorded in the
    # report") goes to a separate timing report when --timings PATH is given.
    if args.timings:
        Path(args.timings).write_text(json.dumps(dict(_provenance(spec, hw), kind="plan-timings", shapes=timings),
                                                 sort_keys=True, indent=1) + "\n")
    if args.emit == "loopnest":
        _write(loopnest_text(doc, args.index), args.out)
    elif args.emit == "csv":
        _write(plan_csv(doc), args.out)
    else:
        _write(json.dumps(doc, sort_keys=True, indent=1) + "\n", args.out)
    return 0


def plan_csv(doc: dict) -> str:
    """One CSV row per (shape, ranked plan) of a plan report (SPEC --emit csv)."""
    cols = ["schema", "descriptor", "workload_hash", "binding", "rank", "tau", "parts", "sia", "est_total_s",
            "padding_fraction"]
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=cols, lineterminator="\n")
    w.writeheader()
    for sh in doc["shapes"]:
        for r, p in enumerate(sh["plans"]):
            w.writerow({"schema": SCHEMA, "descriptor": doc["descriptor"], "workload_hash": doc["workload_hash"],
                        "binding": _binding_key(sh["binding"]), "rank": r, "tau": p["tau"],
                        "parts": " + ".join(f"{q['count']}x{q['smem']}" for q in p["parts"]), "sia": repr(p["sia"]),
                        "est_total_s": repr(p["estimate"]["total_s"]), "padding_fraction": repr(p["padding_fraction"])})
    return buf.getvalue()


def loopnest_text(doc: dict, index: int = 0) -> str:
    """Fig. 8-style tiled loop nest of plan `index` of every shape in a plan
    report: per part, block tiles (x.0) over the covered extents, the k
    staging loop, thread tiles (x.1) and register tiles (x.2)."""
    space, red = doc["axes"]["space"], doc["axes"]["reduce"]
    out = io.StringIO()
    for sh in doc["shapes"]:
        b = sh["binding"]
        if index >= len(sh["plans"]):
            raise E.InputError(f"plan index {index} out of range ({len(sh['plans'])} plans)", field="index")
        plan = sh["plans"][index]
        tau = plan["tau"]
        out.write(f"// {doc['workload']} {_binding_key(b)}: plan {index}, tau={tau}, sia={plan['sia']}, "
                  f"{len(plan['parts'])} part(s)\n")
        off = 0
        for q, part in enumerate(plan["parts"]):
            reg = dict(zip(space, part["reg"]))
            smem = dict(zip(space + red, part["smem"]))
            ext = {}
            for a in space:
                if a == tau:
                    ext[a] = (off, off + part["count"] * smem[a])
                else:
                    e = int(sh["extents"][a])
                    ext[a] = (0, -(-e // smem[a]) * smem[a])
            out.write(f"// part {q}: {part['count']} tile(s) of {tau}={smem[tau]} at {tau} offset {off}\n")
            ind = ""
            for a in space:
                lo, hi = ext[a]
                out.write(f"{ind}for {a}.0 in range({lo}, {hi}, {smem[a]}):  # block tiles\n")
                ind += "  "
            for r in red:
                e = int(sh["extents"][r])
                out.write(f"{ind}for {r}.0 in range(0, {-(-e // smem[r]) * smem[r]}, {smem[r]}):  # stage to shared memory\n")
                ind += "  "
            for a in space:
                out.write(f"{ind}for {a}.1 in range(0, {smem[a]}, {reg[a]}):  # thread tiles\n")
                ind += "  "
            for r in red:
                out.write(f"{ind}for {r}.1 in range({smem[r]}):\n")
                ind += "  "
            for a in space:
                out.write(f"{ind}for {a}.2 in range({reg[a]}):  # register tiles\n")
                ind += "  "
            idx = {a: f"{a}.0 + {a}.1 + {a}.2" for a in space}
            idx.update({r: f"{r}.0 + {r}.1" for r in red})
            ot, oaxes = doc["output"]
            prod = " * ".join(f"{t}[{', '.join(idx[a] for a in axes)}]" for t, axes in doc["inputs"])
            out.write(f"{ind}{ot}[{', '.join(idx[a] for a in oaxes)}] += {prod}\n")
            off += part["count"] * smem[tau]
    return out.getvalue()


def cmd_emit_loopnest(args) -> int:
    if not args.plan:
        raise E.InputError("--plan is required", field="plan")
    p = Path(args.plan)
    if not p.exists():
        raise E.InputError(f"plan file not found: {p}", field="plan")
    doc = json.loads(p.read_text())
    if doc.get("kind") != "plan-report":
        raise E.InputError(f"{p} is not a plan report", field="plan")
    _write(loopnest_text(doc, args.index), args.out)
    return 0


def cmd_sweep(args) -> int:
    """One CSV row per binding: chosen plan, SIA, estimated times, padding,
    occupancy; per-shape errors become status rows (SPEC cmd_sweep)."""
    hw, spec = _hardware(args.hardware), _workload(args.workload)
    coeffs = _coeffs(args.coeffs)
    bindings = _bindings(spec, args.shape, args.range)
    cols = ["schema", "descriptor", "workload_hash", "binding", "status", "error", "relaxation", "candidates",
            "tau", "parts", "sia", "est_total_s", "est_compute_s", "est_memory_s", "est_padding_s", "waves",
            "padding_fraction", "occupancy"]
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=cols, lineterminator="\n")
    w.writeheader()
    prov = _provenance(spec, hw)
    params = _params(args)

    def one(b):
        row = {"schema": SCHEMA, "descriptor": hw.name, "workload_hash": prov["workload_hash"],
               "binding": _binding_key(b)}
        try:  # per-shape errors become status rows; the sweep continues
            inst = WorkloadInstance(spec=spec, bindings=b)
            sec = compile_shape(inst, hw, params)
            row.update(relaxation=sec.relaxation, candidates=len(sec.candidates))
            top = rank_topk(sec.candidates, inst, coeffs=coeffs, k=1)
            d = _plan_doc(top[0], inst, hw, coeffs)
            row.update(status="ok", error="", tau=d["tau"], sia=repr(d["sia"]),
                       parts=" + ".join(f"{p['count']}x{p['smem']}" for p in d["parts"]),
                       est_total_s=repr(d["estimate"]["total_s"]), est_compute_s=repr(d["estimate"]["compute_s"]),
                       est_memory_s=repr(d["estimate"]["memory_s"]), est_padding_s=repr(d["estimate"]["padding_s"]),
                       waves=d["estimate"]["waves"], padding_fraction=repr(d["padding_fraction"]),
                       occupancy=repr(sum(p["occ"] for p in d["parts"]) / len(d["parts"])))
        except E.TunerError as exc:
            row.update(status=type(exc).__name__, error=str(exc))
        return row

    if args.workers > 1 and len(bindings) > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=args.workers) as ex:
            rows = list(ex.map(one, bindings))  # binding order at any worker count
    else:
        rows = [one(b) for b in bindings]
    for row in rows:
        w.writerow(row)
    _write(buf.getvalue(), args.out)
    return 0


# ---------------------------------------------------------------- entry point

def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2407_21418_b200.cli", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p, workload=True):
        if workload:
            p.add_argument("--workload")
            p.add_argument("--hardware")
            p.add_argument("--shape", action="append")
            p.add_argument("--range", action="append")
            p.add_argument("--psi", type=float)
            p.add_argument("--coeffs")
            p.add_argument("--workers", type=int)
        p.add_argument("--out")

    common(sub.add_parser("tune", help="compile stage -> candidate cache"))
    p = sub.add_parser("plan", help="combine + SIA Top-K -> plan report")
    common(p)
    p.add_argument("--cache")
    p.add_argument("--topk", type=int)
    p.add_argument("--emit", choices=["plan", "loopnest", "csv"])
    p.add_argument("--index", type=int)
    p.add_argument("--timings", help="write combine + rank wall-clock to this file (keeps the plan report "
                                     "byte-identical across runs)")
    p = sub.add_parser("emit-loopnest", help="plan report -> tiled loop nest text")
    common(p, workload=False)
    p.add_argument("--plan")
    p.add_argument("--index", type=int)
    common(sub.add_parser("sweep", help="per-shape CSV over a range"))
    return ap


# Flag defaults, applied AFTER the FTB_CLI_* environment overrides: a flag
# given on the command line wins, then the environment, then these.
DEFAULTS = {"workers": 1, "topk": 10, "emit": "plan", "index": 0}


def _env_defaults(args) -> None:
    for k, v in vars(args).items():
        if v is None or v == []:
            env = os.environ.get("FTB_CLI_" + k.upper())
            if env is not None:
                setattr(args, k, env.split(";") if k in ("shape", "range") else
                        (int(env) if k in ("topk", "index", "workers") else (float(env) if k == "psi" else env)))
            elif k in DEFAULTS:
                setattr(args, k, DEFAULTS[k])
    if getattr(args, "emit", None) not in (None, "plan", "loopnest", "csv"):
        raise ValueError(f"--emit / FTB_CLI_EMIT must be plan, loopnest or csv, not {args.emit!r}")


def main(argv: list[str] | None = None) -> int:
    args = _parser().parse_args(argv)
    _env_defaults(args)
    cmds = {"tune": cmd_tune, "plan": cmd_plan, "emit-loopnest": cmd_emit_loopnest, "sweep": cmd_sweep}
    try:
        return cmds[args.cmd](args)
    except E.TunerError as exc:
        print(f"error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return exc.exit_code
    except (OSError, ValueError, KeyError) as exc:
        print(f"error: InputError: {exc}", file=sys.stderr)
        return E.EXIT_INPUT
    except Exception as exc:  # invariant violations and bugs: exit 3, never a traceback-only crash
        print(f"error: InternalError: {type(exc).__name__}: {exc}", file=sys.stderr)
        return E.EXIT_INTERNAL


if __name__ == "__main__":
    sys.exit(main())
