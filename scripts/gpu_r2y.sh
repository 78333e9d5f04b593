SHAPES="bmm 384 46 46 64 nk" NL=4 COLD=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:ftb_tc -s 6 -c 1 -o /tmp/bmm46 -f python scripts/chain_time.py > /tmp/ncu.log 2>&1; echo rc=$?
ncu -i /tmp/bmm46.ncu-rep --page source --csv --print-source sass > gpurun_out/r2y_bmm46_source.csv 2>/dev/null; echo rc2=$?
ncu -i /tmp/bmm46.ncu-rep --page details --csv > gpurun_out/r2y_bmm46_details.csv 2>/dev/null
ls -la gpurun_out/
