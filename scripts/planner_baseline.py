"""Tuning time, reference vs this repo, on the same shapes and descriptor
(SURVEY §8(d) CPU baseline (i)): the reference's compile_shape +
build_programs + rank_programs (single Python process, 1 core, per-shape
wall-clock cap) against the C++ planner (1 thread), B200 bf16 parity-mode
descriptor. Top-1 plans are compared for identity. Needs /root/reference
(this container only). Writes profiles/r1_planner_vs_reference.json."""
import json, os, subprocess, sys, time
sys.path.insert(0, ".")
CAP = float(os.environ.get("CAP_S", "120"))
REF = "/root/reference/pkg/src"
CHILD = r'''
import json, sys, time
from mktune.hardware import load_hardware_descriptor
from mktune.workload import parse_workload, WorkloadInstance
from mktune.filtering import compile_shape
from mktune.combine import build_programs
from mktune.scoring import rank_programs
hw = load_hardware_descriptor(sys.argv[1]); spec = parse_workload(sys.argv[2]); b = json.loads(sys.argv[3])
inst = WorkloadInstance(spec=spec, bindings=b)
t0 = time.perf_counter(); res = compile_shape(inst, hw); t1 = time.perf_counter()
pool = build_programs(res.candidates, inst); t2 = time.perf_counter()
top = rank_programs(pool, k=10); t3 = time.perf_counter()
p = top[0]
print(json.dumps({"compile_s": t1 - t0, "build_s": t2 - t1, "rank_s": t3 - t2, "pool": len(pool),
                  "top1": [[sorted(k.smem_tile.items()), n] for k, n in p.parts], "sia": p.sia}))
'''


def main():
    from paper_2407_21418_b200.mktune.hardware import b200_bf16, serialize_hardware_descriptor
    from paper_2407_21418_b200.runtime import Planner
    from paper_2407_21418_b200.workloads import bert_layer_shapes
    hw = b200_bf16(tcgen05=False)
    hw_doc = serialize_hardware_descriptor(hw)
    shapes = [s for T in (5, 38, 62, 128) for s in bert_layer_shapes(T) if s.name in ("qkv", "ffn2", "scores")]
    pl = Planner(hw=hw, threads=1)
    rows = []
    for sh in shapes:
        inst = sh.instance()
        t0 = time.perf_counter()
        rec = pl.plan([inst])[0]
        ours = time.perf_counter() - t0
        d = rec.describe()
        row = {"shape": f"{sh.name} b{sh.batch} M{sh.M} N{sh.N} K{sh.K}", "ours_s": ours, "ours_top1_sia": d["sia"]}
        env = dict(os.environ, PYTHONPATH=REF, PYTHONDONTWRITEBYTECODE="1")
        try:
            t0 = time.perf_counter()
            out = subprocess.run([sys.executable, "-c", CHILD, hw_doc, json.dumps(inst.spec.to_doc()),
                                  json.dumps(dict(inst.bindings))], env=env, capture_output=True, text=True,
                                 timeout=CAP, cwd="/tmp")
            wall = time.perf_counter() - t0
            if out.returncode != 0:
                row["reference"] = {"error": out.stderr.strip().splitlines()[-1][:200]}
            else:
                r = json.loads(out.stdout.strip().splitlines()[-1])
                r["wall_s"] = wall
                r["same_top1_sia"] = abs(r["sia"] - d["sia"]) == 0.0
                row["reference"] = r
                row["speedup"] = (r["compile_s"] + r["build_s"] + r["rank_s"]) / ours
        except subprocess.TimeoutExpired:
            row["reference"] = {"timeout_s": CAP}
            row["speedup_at_least"] = CAP / ours
        print(json.dumps(row), flush=True)
        rows.append(row)
    doc = {"what": "tuning time per shape: reference mktune (compile_shape + build_programs + rank_programs, "
                   "1 Python process) vs the C++ planner (1 thread), B200 bf16 parity-mode descriptor",
           "cap_s": CAP, "host_cpus": os.cpu_count(), "rows": rows}
    json.dump(doc, open("profiles/r1_planner_vs_reference.json", "w"), indent=1)


if __name__ == "__main__":
    main()
