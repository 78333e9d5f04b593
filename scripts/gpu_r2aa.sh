timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
timeout 1500 python bench.py --steps 5 --warmup 3 --c4-shapes 0 --dynamic-steps 0 --no-cpu --per-shape-rows > gpurun_out/r2aa_bench.json 2> gpurun_out/r2aa_bench.err; echo bench_rc=$?
tail -3 gpurun_out/r2aa_bench.err
