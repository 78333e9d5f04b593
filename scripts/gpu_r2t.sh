M=$(python scripts/ncu_shapes.py metrics)
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2t_ncu_shapes.csv python scripts/ncu_shapes.py run --manifest gpurun_out/r2t_manifest.json > gpurun_out/r2t_ncu.log 2>&1; echo ncu_rc=$?
tail -5 gpurun_out/r2t_ncu.log
ls -la gpurun_out/
