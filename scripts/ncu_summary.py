"""Summarise an ncu report (--set full) into markdown: per kernel the
duration, DRAM bytes, L2->SM bytes, tensor-pipe activity and top stalls.
usage: python scripts/ncu_summary.py REPORT.ncu-rep [title] > profiles/X.md"""
import csv, io, subprocess, sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM bytes"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "tc pipe active % (elapsed)"),
    ("smsp__sass_inst_executed_op_utcmma.sum", "UTCMMA instructions"),
    ("smsp__sass_inst_executed_op_tmem_ldt.sum", "tcgen05.ld instructions"),
    ("launch__grid_size", "grid"),
    ("launch__cluster_dim_x", "cluster x"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
]
print(f"# ncu summary: {title}\n")
print(f"source report: `{rep}` (ncu --set full --clock-control none)\n")
for row in rows[2:]:
    d = dict(zip(hdr, row))
    u = dict(zip(hdr, units))
    print(f"## {d.get('Kernel Name','?')[:90]}\n")
    print("| metric | value | unit |\n|---|---|---|")
    for k, name in keys:
        if k in d and d[k] not in ("", "n/a"):
            print(f"| {name} (`{k}`) | {d[k]} | {u.get(k,'')} |")
    stalls = []
    for k in hdr:
        if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio") or \
           k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(d[k]), k))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    if stalls:
        print("\ntop warp stall reasons (per issue active):\n")
        for v, k in stalls[:6]:
            print(f"- `{k}`: {v:.2f}")
    print()
