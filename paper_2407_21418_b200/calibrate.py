"""On-device SIA calibration (the paper's §6.3 analog,
PAPER.md:515, :636-638): how well does the analytic SIA ranking
(scoring.py:23-126) predict measured B200 time, and which score coefficients
make the planner pick the fastest plans?

* `topk_regret`: per shape, the SIA Top-k plans (B200 legality mode) are each
  timed alone (CUDA graph of back-to-back launches); reports the measured rank
  of SIA's top-1 and time(top-1) / time(best of the Top-k).
* `coeff_sweep`: for a grid of `SiaCoeffs`, plan the shape set (full fallback
  ladder) and time it both per shape and as one grouped table.

    python -m paper_2407_21418_b200.calibrate --out profiles/r1_sia_calibration.json

Needs a B200 (the timings are the point); planning alone runs anywhere.
"""

from __future__ import annotations

import argparse
import json
import time


def _bind(shape, device, seed=0):
    import torch

    g = torch.Generator(device=device).manual_seed(seed)

    def rnd(*s):
        return (torch.rand(*s, generator=g, device=device) * 2 - 1).bfloat16()

    if shape.kind == "dense":
        A = rnd(shape.M, shape.K)
        B = rnd(shape.N, shape.K) if shape.b_layout == "nk" else rnd(shape.K, shape.N)
        C = torch.empty(shape.M, shape.N, dtype=torch.bfloat16, device=device)
        return A, B, C
    kp = (shape.K + 7) // 8 * 8
    A = rnd(shape.batch, shape.M, kp)[:, :, : shape.K]
    B = rnd(shape.batch, shape.N, shape.K) if shape.b_layout == "nk" else rnd(shape.batch, shape.K, shape.N)
    npad = (shape.N + 7) // 8 * 8
    C = torch.empty(shape.batch, shape.M, npad, dtype=torch.bfloat16, device=device)[:, :, : shape.N]
    return A, B, C


def time_launches(launch, reps: int = 10, rounds: int = 3) -> float:
    """Microseconds per launch: `reps` launches captured in a CUDA graph, best of `rounds`."""
    import torch

    # launches of one table must not overlap each other (the split-K workspace
    # and its counters are per table): drain earlier work on other streams first
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        launch(s)
        launch(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            launch(s)
    best = float("inf")
    for _ in range(rounds):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def topk_regret(shapes, k: int = 5, device="cuda") -> list[dict]:
    from .execute import Executable, gemm_desc, program_from_plan
    from .mktune.errors import EmptyResultError
    from .mktune.filtering import compile_shape
    from .mktune.hardware import b200_bf16
    from .mktune.scoring import rank_topk

    hw = b200_bf16(tcgen05=True)
    rows = []
    for sh in shapes:
        inst = sh.instance()
        try:
            plans = rank_topk(compile_shape(inst, hw).candidates, inst, k=k)
        except EmptyResultError:
            rows.append({"shape": _name(sh), "skipped": "no strict-legal tau cover (fallback ladder shape)"})
            continue
        A, B, C = _bind(sh, device)
        times = []
        for p in plans:
            ex = Executable([gemm_desc(A, B, C, sh.b_layout)], [program_from_plan(p)], (A, B, C))
            times.append(time_launches(lambda s, ex=ex: ex.launch(s)))
            ex.close()
        best = min(range(len(times)), key=times.__getitem__)
        rows.append({"shape": _name(sh), "us": times, "sia": [p.sia for p in plans],
                     "best_rank": best, "top1_over_best": times[0] / times[best]})
    return rows


def coeff_sweep(shapes, grid, device="cuda") -> list[dict]:
    import torch

    from .execute import Executable, gemm_desc
    from .mktune.scoring import SiaCoeffs
    from .runtime import Planner

    bound = [_bind(sh, device, seed=i) for i, sh in enumerate(shapes)]
    flops = sum(s.flops for s in shapes)
    out = []
    for c in grid:
        pl = Planner(coeffs=SiaCoeffs(*c))
        t0 = time.perf_counter()
        recs = pl.plan([s.instance() for s in shapes])
        tune = time.perf_counter() - t0
        per_shape = 0.0
        for (A, B, C), sh, r in zip(bound, shapes, recs):
            ex = Executable([gemm_desc(A, B, C, sh.b_layout)], [r.program], (A, B, C))
            per_shape += time_launches(lambda s, ex=ex: ex.launch(s))
            ex.close()
        descs = [gemm_desc(A, B, C, sh.b_layout) for (A, B, C), sh in zip(bound, shapes)]
        grouped = Executable(descs, [r.program for r in recs], [t for b in bound for t in b])
        g_us = time_launches(lambda s: grouped.launch(s), reps=5)
        grouped.close()
        torch.cuda.synchronize()
        out.append({"coeffs": list(c), "per_shape_sum_us": per_shape, "grouped_us": g_us,
                    "grouped_tflops": flops / (g_us * 1e-6) / 1e12, "tuning_s": tune})
    return out


def spearman(x, y) -> float:
    """Spearman rank correlation (average ranks for ties); nan if degenerate."""
    import numpy as np

    def ranks(v):
        v = np.asarray(v, dtype=np.float64)
        order = v.argsort(kind="mergesort")
        r = np.empty(len(v))
        r[order] = np.arange(len(v), dtype=np.float64)
        for val in np.unique(v):  # ties share their mean rank
            m = v == val
            r[m] = r[m].mean()
        return r

    if len(x) < 3:
        return float("nan")
    a, b = ranks(x), ranks(y)
    if a.std() == 0 or b.std() == 0:
        return float("nan")
    return float(np.corrcoef(a, b)[0, 1])


def model_vs_measured(shapes, device="cuda") -> dict:
    """f-2 / oracles.exhaustive_rank_check in spirit (oracles.py:96-122,
    timemodel.py:56-123): for every shape the runtime's Top-1 plan is timed
    alone on the device and compared with the analytic estimate_time of that
    plan (B200 descriptor). Reports per-shape rows and the Spearman rank
    correlation of estimated vs measured time over the shape set."""
    from .execute import Executable, gemm_desc
    from .mktune.combine import ProgramPlan  # noqa: F401  (type of the plans estimate_time reads)
    from .mktune.hardware import b200_bf16
    from .mktune.timemodel import estimate_time
    from .runtime import Planner

    hw = b200_bf16(tcgen05=True)
    pl = Planner()
    recs = pl.plan([s.instance() for s in shapes])
    rows = []
    for sh, r in zip(shapes, recs):
        A, B, C = _bind(sh, device)
        ex = Executable([gemm_desc(A, B, C, sh.b_layout)], [r.program], (A, B, C))
        us = time_launches(lambda s, ex=ex: ex.launch(s))
        ex.close()
        est = estimate_time(_plan_of(r.program, sh.instance()), sh.instance(), hw)
        rows.append({"shape": _name(sh), "measured_us": us, "estimate_us": est.total_s * 1e6,
                     "stage": r.stage, "sia": r.program.sia})
    return {"rows": rows,
            "spearman_estimate_vs_measured": spearman([x["estimate_us"] for x in rows], [x["measured_us"] for x in rows]),
            "median_measured_over_estimate": sorted(x["measured_us"] / x["estimate_us"] for x in rows)[len(rows) // 2]}


def rank_spread(shapes, k: int = 400, picks: int = 8, device="cuda") -> dict:
    """Within one shape, does SIA order plans like the device does? The
    strict-legal pool's Top-k (k=400) is ranked by SIA; `picks` plans at
    evenly spaced ranks are timed; per shape the Spearman correlation of SIA
    rank vs measured time and of estimate_time vs measured time (ties in the
    SIA score are the norm — SURVEY §7.3 — so ranks, not scores, are used)."""
    from .execute import Executable, gemm_desc, program_from_plan
    from .mktune.errors import EmptyResultError
    from .mktune.filtering import compile_shape
    from .mktune.hardware import b200_bf16
    from .mktune.scoring import rank_topk
    from .mktune.timemodel import estimate_time

    hw = b200_bf16(tcgen05=True)
    rows = []
    for sh in shapes:
        inst = sh.instance()
        try:
            plans = rank_topk(compile_shape(inst, hw).candidates, inst, k=k)
        except EmptyResultError:
            rows.append({"shape": _name(sh), "skipped": "no strict-legal cover of the main axis (fallback rung shape)"})
            continue
        idx = sorted({round(i * (len(plans) - 1) / max(1, picks - 1)) for i in range(picks)})
        A, B, C = _bind(sh, device)
        us, est = [], []
        for i in idx:
            ex = Executable([gemm_desc(A, B, C, sh.b_layout)], [program_from_plan(plans[i])], (A, B, C))
            us.append(time_launches(lambda s, ex=ex: ex.launch(s)))
            ex.close()
            est.append(estimate_time(plans[i], inst, hw).total_s * 1e6)
        rows.append({"shape": _name(sh), "ranks": idx, "us": us, "estimate_us": est,
                     "sia": [plans[i].sia for i in idx], "rho_rank": spearman(idx, us),
                     "rho_estimate": spearman(est, us), "top1_over_best": us[0] / min(us)})
    done = [r for r in rows if "rho_rank" in r]
    import math

    def mean(v):
        v = [x for x in v if not math.isnan(x)]
        return sum(v) / len(v) if v else float("nan")

    return {"rows": rows, "mean_rho_sia_rank_vs_measured": mean([r["rho_rank"] for r in done]),
            "mean_rho_estimate_vs_measured": mean([r["rho_estimate"] for r in done]),
            "top1_within_10pct_of_best_sampled": sum(r["top1_over_best"] <= 1.10 for r in done), "shapes": len(done)}


def _plan_of(program, inst):
    """A facade ProgramPlan from an ftb_program (for estimate_time)."""
    from .mktune.combine import ProgramPlan
    from .mktune.ukernel import UKernel

    spec = inst.spec
    space, axes = list(spec.space_axes), list(spec.space_axes) + list(spec.reduce_axes)
    parts = []
    for p in range(program.n_parts):
        k = UKernel(reg_tile={a: int(program.reg[p][i]) for i, a in enumerate(space)},
                    smem_tile={a: int(program.smem[p][i]) for i, a in enumerate(axes)})
        parts.append((k, int(program.count[p])))
    return ProgramPlan(parts=tuple(parts), tau=space[program.tau], shape=inst, sia=program.sia)


def _name(sh) -> str:
    return f"{sh.name} b{sh.batch} M{sh.M} N{sh.N} K{sh.K}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--r2", action="store_true", help="round-2 calibration (model vs measured, rank spread, A/B)")
    args = ap.parse_args()
    from .workloads import CANONICAL_T, bert_layer_shapes, c1_shapes

    canon = [s for T in CANONICAL_T for s in bert_layer_shapes(T)]
    grid = [(1.0, 1.0, 1.0), (1.0, 1.0, 0.25), (2.0, 1.0, 0.5), (4.0, 1.0, 0.25), (1.0, 1.0, 0.0), (1.0, 0.0, 0.0),
            (1.0, 0.5, 1.0), (0.5, 1.0, 1.0)]
    if args.r2:
        # round 2: the final kernel; estimate_time vs measured
        # over all 192 bench shapes, SIA-rank spread per canonical shape, and the
        # A/B of the coefficient candidate (0.5, 1, 1) against the default
        bench = c1_shapes(24, 0)
        res = {
            "what": "r2 SIA calibration on the final kernel (L2-warm CUDA-graph timing per plan)",
            "model_vs_measured": model_vs_measured(bench),
            "rank_spread": rank_spread(canon),
            "coeff_ab": coeff_sweep(bench, [(1.0, 1.0, 1.0), (0.5, 1.0, 1.0)]),
        }
        ab = res["coeff_ab"]
        res["summary"] = {
            "spearman_estimate_vs_measured_192": res["model_vs_measured"]["spearman_estimate_vs_measured"],
            "mean_rho_sia_rank_vs_measured": res["rank_spread"]["mean_rho_sia_rank_vs_measured"],
            "mean_rho_estimate_vs_measured_within_shape": res["rank_spread"]["mean_rho_estimate_vs_measured"],
            "default_per_shape_sum_us": ab[0]["per_shape_sum_us"], "c050_per_shape_sum_us": ab[1]["per_shape_sum_us"],
            "default_grouped_us": ab[0]["grouped_us"], "c050_grouped_us": ab[1]["grouped_us"],
        }
        text = json.dumps(res, indent=1)
        if args.out:
            open(args.out, "w").write(text + "\n")
        print(json.dumps(res["summary"]))
        return
    res = {
        "what": "SIA Top-k regret per C1 canonical shape and a SiaCoeffs grid timed per shape and grouped (C1, 192 shapes)",
        "topk_regret": topk_regret(canon, k=args.k),
        "coeff_sweep": coeff_sweep(c1_shapes(24, 0), grid),
    }
    reg = [r for r in res["topk_regret"] if "top1_over_best" in r]
    if reg:
        res["summary"] = {
            "shapes_ranked": len(reg),
            "top1_is_best": sum(r["best_rank"] == 0 for r in reg),
            "mean_top1_over_best": sum(r["top1_over_best"] for r in reg) / len(reg),
            "best_coeffs_grouped": min(res["coeff_sweep"], key=lambda r: r["grouped_us"])["coeffs"],
            "best_coeffs_per_shape": min(res["coeff_sweep"], key=lambda r: r["per_shape_sum_us"])["coeffs"],
        }
    text = json.dumps(res, indent=1)
    if args.out:
        open(args.out, "w").write(text + "\n")
    print(json.dumps(res.get("summary", {})))


if __name__ == "__main__":
    main()
