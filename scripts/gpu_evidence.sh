# Full evidence pass: tests, smoke, bench (default), reference arm, ncu launch list + full capture.
export PYTHONUNBUFFERED=1
TAG=${TAG:-r1}
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2 | tee gpurun_out/smoke_$TAG.txt
timeout 500 python bench.py --per-shape-rows > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -c 600 gpurun_out/bench_$TAG.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; tail -c 300 gpurun_out/bench_ref_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ftb -c 40 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --min-warm-s 0 --per-shape 0 --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; tail -1 gpurun_out/ncu_launch_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ftb -s 4 -c 1 -o gpurun_out/prof_step_$TAG python bench.py --steps 3 --warmup 3 --min-warm-s 0 --per-shape 0 --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1; tail -1 gpurun_out/ncu_full_$TAG.log
