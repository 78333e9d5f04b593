set -x
python __graft_entry__.py smoke 2>&1 | tail -8
timeout 300 python bench.py --steps 20 --warmup 5 --per-shape-rows > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err
head -c 3000 gpurun_out/bench1.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 3 --warmup 3 --per-shape 0 --no-cpu --min-warm-s 0 > /dev/null 2>&1
grep -c ftb gpurun_out/launches_r1.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ftb_tc -s 4 -c 1 -o gpurun_out/prof_r1 python bench.py --steps 2 --warmup 3 --per-shape 0 --no-cpu --min-warm-s 0 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
