set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/r2a_pytest_gpu.txt 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2a_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.txt 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/r2a_smoke.txt
timeout 1200 python bench.py --steps 5 --warmup 3 --per-shape-rows > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r2a_bench.json; tail -20 gpurun_out/r2a_bench.err
