M=$(python scripts/ncu_shapes.py metrics)
timeout 1500 ncu --metrics $M --clock-control none --cache-control none -k regex:ftb_ --csv --log-file gpurun_out/r2u_ncu_shapes.csv python scripts/ncu_shapes.py run --manifest gpurun_out/r2u_manifest.json > gpurun_out/r2u_ncu.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/r2u_ncu.log
