# final-build ncu evidence: per-shape counters + traffic artefact, launch list of the default bench, --set full of the grouped step
M=$(python scripts/ncu_shapes.py metrics)
timeout 1500 ncu --metrics $M --clock-control none --cache-control none -k regex:ftb_ --csv --log-file gpurun_out/r2bl_ncu_shapes.csv python scripts/ncu_shapes.py run --manifest gpurun_out/r2bl_manifest.json > gpurun_out/r2bl_ncu.log 2>&1; echo ncu_shapes_rc=$?
tail -2 gpurun_out/r2bl_ncu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ftb -c 400 --csv --log-file gpurun_out/r2bl_launches.csv python bench.py --steps 2 --warmup 3 --min-warm-s 0 --no-cpu --dynamic-steps 0 --c4-shapes 64 --tuning-budget-s 2 > gpurun_out/r2bl_launch.log 2>&1; echo launches_rc=$?
tail -2 gpurun_out/r2bl_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ftb_tc -s 2 -c 1 -o /tmp/r2bl_step python scripts/step_once.py > gpurun_out/r2bl_full.log 2>&1; echo full_rc=$?
python scripts/ncu_summary.py /tmp/r2bl_step.ncu-rep "C1 grouped step, round 2 final build" > gpurun_out/r2bl_ncu_step.md 2>&1; echo summary_rc=$?
ncu -i /tmp/r2bl_step.ncu-rep --page raw --csv > gpurun_out/r2bl_step_raw.csv 2>/dev/null; ls -la gpurun_out/r2bl_*
