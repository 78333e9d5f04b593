i=0
for S in "dense 608 768 768" "dense 160 768 3072" "bmm 384 100 100 64 nk" "dense 128 256 64" "bmm 384 5 5 64 nk"; do
  i=$((i+1))
  SHAPES="$S" NL=4 timeout 300 ncu --set full --clock-control none -k regex:ftb_tc -s 2 -c 1 -o /tmp/r2f_shape$i -f python scripts/chain_time.py > /tmp/r2f_ncu$i.log 2>&1
  echo "$S -> $?"
  ncu -i /tmp/r2f_shape$i.ncu-rep --page details --csv > gpurun_out/r2f_details$i.csv 2>/dev/null
  ncu -i /tmp/r2f_shape$i.ncu-rep --page raw --csv > gpurun_out/r2f_raw$i.csv 2>/dev/null
done
ls -la gpurun_out
