timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2p_pytest.txt 2>&1; tail -3 gpurun_out/r2p_pytest.txt
timeout 1200 python bench.py --steps 5 --warmup 3 --per-shape-rows > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err; echo bench_rc=$?
tail -3 gpurun_out/r2p_bench.err
