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


def _name(sh) -> str:
    return f"{sh.name} b{sh.batch} M{sh.M} N{sh.N} K{sh.K}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--k", type=int, default=5)
    args = ap.parse_args()
    from .workloads import CANONICAL_T, bert_layer_shapes, c1_shapes

    canon = [s for T in CANONICAL_T for s in bert_layer_shapes(T)]
    grid = [(1.0, 1.0, 1.0), (1.0, 1.0, 0.25), (2.0, 1.0, 0.5), (4.0, 1.0, 0.25), (1.0, 1.0, 0.0), (1.0, 0.0, 0.0),
            (1.0, 0.5, 1.0), (0.5, 1.0, 1.0)]
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
