"""Per-shape ncu evidence (north_star: "ncu counters (tensor-pipe utilisation;
achieved HBM GB/s for skinny small-M shapes) must show each shape's
throughput against min(dense bf16 tensor peak, HBM bytes at 8 TB/s)").

Two modes:
  run    (under ncu, on the GPU box): every shape of the C1 bench set, C3 M in
         {1,16,64,127,256,1000,4096} and C2 T in {1,64,257,512} (scores and
         context) is planned and lowered to its own single-problem table and
         launched twice (warm, then profiled), then the grouped C1 step table
         twice; the launch order is written to --manifest.
  report (anywhere): joins ncu's CSV (--metrics ... --csv --log-file) with the
         manifest -> profiles/<tag>_ncu_shapes.md (+ .json) and the per-build
         traffic artefact profiles/ncu_traffic.json that bench.py reads
         (keyed by the sha256 of libftb.so).

  ncu --metrics $(python scripts/ncu_shapes.py metrics) --clock-control none --cache-control none \
      -k regex:ftb_ --csv --log-file gpurun_out/ncu_shapes.csv python scripts/ncu_shapes.py run --manifest gpurun_out/ncu_manifest.json
  python scripts/ncu_shapes.py report gpurun_out/ncu_shapes.csv gpurun_out/ncu_manifest.json r2
The profiled (second) launch of every shape follows a 256 MB buffer write
(2x L2), so its operands are L2-cold as in bench.py's per-shape timing;
ncu's own cache flush is off (--cache-control none), which would also empty
the instruction cache and add ~9 us to every small launch (r2t).
"""
import csv
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

STALLS = ["long_scoreboard", "wait", "barrier", "membar", "sleeping", "short_scoreboard", "no_instruction",
          "math_pipe_throttle", "lg_throttle", "mio_throttle", "dispatch_stall", "branch_resolving", "selected"]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__cycles_elapsed.avg.per_second"] + [
    f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in STALLS]


def shapes():
    from paper_2407_21418_b200.workloads import Shape, c1_shapes

    out = [("c1", s) for s in c1_shapes(24, 0)]
    out += [("c3", Shape("dense", "llm", 1, m, 4096, 4096, "nk")) for m in (1, 16, 64, 127, 256, 1000, 4096)]
    for T in (1, 64, 257, 512):
        out.append(("c2", Shape("bmm", "scores", 1024, T, T, 64, "nk", ("i", "j"))))
        out.append(("c2", Shape("bmm", "context", 1024, T, 64, T, "kn", ("i", "k"))))
    return out


def run(manifest: str):
    import torch

    from paper_2407_21418_b200.execute import Executable, gemm_desc
    from paper_2407_21418_b200.runtime import Planner
    from paper_2407_21418_b200.shapeset import ShapeSet

    planner = Planner()
    todo = shapes()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")  # 2x L2: evicts every operand
    order = []
    for i in range(0, len(todo), 48):  # bounded memory: 48 shapes bound at a time
        chunk = todo[i:i + 48]
        ss = ShapeSet([s for _, s in chunk], planner, device="cuda:0", seed=i)
        for (cfg, s), x, rec in zip(chunk, ss.bound, ss.records):
            ex = Executable([gemm_desc(x.A, x.B, x.C, s.b_layout)], [rec.program])
            ex.launch()
            flush.fill_(1)
            ex.launch()
            torch.cuda.synchronize()
            order.append({"cfg": cfg, "name": s.name, "b": s.batch, "M": s.M, "N": s.N, "K": s.K,
                          "flops": s.flops, "bytes": s.bytes, "launches": 2})
            ex.close()
        del ss
    from paper_2407_21418_b200.workloads import c1_shapes

    ss = ShapeSet(c1_shapes(24, 0), planner, device="cuda:0", seed=0)
    ss.launch()
    flush.fill_(2)
    ss.launch()
    torch.cuda.synchronize()
    order.append({"cfg": "c1_step", "name": "grouped C1 step (192 GEMMs, one launch)", "b": 0, "M": 0, "N": 0, "K": 0,
                  "flops": ss.true_flops, "bytes": ss.alg_bytes, "launches": 2})
    Path(manifest).write_text(json.dumps(order))


def _parse(csv_path):
    """ncu --csv --log-file rows -> list of {metric: value} per kernel launch."""
    lines = Path(csv_path).read_text().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rd = csv.DictReader(lines[start:])
    per = {}
    for r in rd:
        if "ftb_" not in r.get("Kernel Name", ""):
            continue
        k = int(r["ID"])
        d = per.setdefault(k, {"kernel": r["Kernel Name"]})
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
                 "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3, "Ghz": 1, "hz": 1e-9, "Mhz": 1e-3}.get(unit, 1)
        d[r["Metric Name"]] = v * scale
    return [per[k] for k in sorted(per)]


def report(csv_path, manifest, tag):
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    P = peaks.get("bf16_tflops", 1679.2) * 1e12
    launches = _parse(csv_path)
    order = json.loads(Path(manifest).read_text())
    rows, i = [], 0
    for o in order:
        got = launches[i:i + o["launches"]]
        i += o["launches"]
        m = got[-1]  # the second (profiled-warm) launch; caches flushed by ncu either way
        us = m["gpu__time_duration.sum"]
        dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        t_roof = max(o["flops"] / P, o["bytes"] / 8e12)
        stalls = sorted(((m.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio", 0.0), s)
                         for s in STALLS), reverse=True)
        rows.append({**o, "ncu_us": us, "dram_bytes": dram, "dram_over_alg": dram / max(1, o["bytes"]),
                     "achieved_dram_gbs": dram / (us * 1e-6) / 1e9, "alg_gbs": o["bytes"] / (us * 1e-6) / 1e9,
                     "tflops": o["flops"] / (us * 1e-6) / 1e12, "roofline_frac_ncu": t_roof / (us * 1e-6),
                     "dram_pct": m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "tensor_pct": m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                     "l2_hit_pct": m.get("lts__t_sector_hit_rate.pct"), "sm_ghz": m.get("sm__cycles_elapsed.avg.per_second"),
                     "top_stalls": [(s, round(v, 2)) for v, s in stalls[:3]], "kernel": m["kernel"][:60]})
    from bench import lib_sha  # the same source hash bench.py checks

    sha = lib_sha()
    c1 = [r for r in rows if r["cfg"] == "c1"]
    step = next(r for r in rows if r["cfg"] == "c1_step")
    traffic = {
        "c1_step": {"lib_sha": sha, "dram_bytes_per_launch": step["dram_bytes"], "how": f"{tag}: ncu, grouped C1 step"},
        "c1_per_shape": {"lib_sha": sha, "dram_bytes_per_launch": sum(r["dram_bytes"] for r in c1),
                         "how": f"{tag}: ncu, sum over the 192 per-shape launches (one each, L2 flushed)"},
    }
    (ROOT / "profiles" / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
    (ROOT / "profiles" / f"{tag}_ncu_shapes.json").write_text(json.dumps(rows, indent=1) + "\n")
    lines = [f"# Per-shape ncu counters ({tag}, libftb.so {sha})", "",
             "Each shape is its own launch (single-problem table), profiled by `ncu --clock-control none",
             "--cache-control none` after a 256 MB L2-evicting write (operands L2-cold, instruction cache warm).",
             "`ncu_us` is ncu's serialised single-launch duration (no PDL overlap with a neighbour launch, so",
             "it is longer than the CUDA-graph chain bench.py times); the counters are the evidence.",
             "roofline = max(F / MEASURED_PEAKS bf16, algorithmic bytes / 8 TB/s).", "",
             "| cfg | op | b | M | N | K | ncu us | TFLOP/s | roof frac | DRAM MB (x alg) | DRAM GB/s | DRAM % | tensor % | L2 hit % | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['cfg']} | {r['name']} | {r['b']} | {r['M']} | {r['N']} | {r['K']} | {r['ncu_us']:.2f} | "
                     f"{r['tflops']:.1f} | {r['roofline_frac_ncu']:.3f} | {r['dram_bytes'] / 1e6:.2f} ({r['dram_over_alg']:.2f}) | "
                     f"{r['achieved_dram_gbs']:.0f} | {r['dram_pct'] or 0:.1f} | {r['tensor_pct'] or 0:.1f} | "
                     f"{r['l2_hit_pct'] or 0:.1f} | {', '.join(f'{s} {v}' for s, v in r['top_stalls'])} |")
    (ROOT / "profiles" / f"{tag}_ncu_shapes.md").write_text("\n".join(lines) + "\n")
    print(f"{len(rows)} rows; c1_step dram {step['dram_bytes'] / 1e9:.3f} GB; lib {sha}")


if __name__ == "__main__":
    if sys.argv[1] == "metrics":
        print(",".join(METRICS))
    elif sys.argv[1] == "run":
        run(sys.argv[sys.argv.index("--manifest") + 1])
    else:
        report(sys.argv[2], sys.argv[3], sys.argv[4])
