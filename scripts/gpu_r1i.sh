# Round-1 re-entry: tests, smoke, bench, ncu launch list + full capture of the step kernels.
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tee gpurun_out/gpu.txt
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
timeout 400 python bench.py --per-shape-rows > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -c 800 gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --min-warm-s 0 --per-shape 0 --no-cpu > gpurun_out/ncu_launch.log 2>&1; tail -3 gpurun_out/ncu_launch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ftb_tc -s 4 -c 2 -o gpurun_out/prof_step python bench.py --steps 3 --warmup 3 --min-warm-s 0 --per-shape 0 --no-cpu > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
