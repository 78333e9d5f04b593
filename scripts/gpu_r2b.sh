timeout 1200 python bench.py --steps 5 --warmup 3 --per-shape-rows > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench_rc=$?
tail -20 gpurun_out/r2b_bench.err
