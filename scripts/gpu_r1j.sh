export PYTHONUNBUFFERED=1
for p in 0 1; do FTB_PAIR=$p timeout 200 python scripts/gemm_probe.py 2>&1 | tail -12; done
timeout 120 python scripts/kb_probe.py 2>&1 | tail -20
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ftb -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --min-warm-s 0 --per-shape 0 --no-cpu > gpurun_out/ncu_launch.log 2>&1; tail -3 gpurun_out/ncu_launch.log
