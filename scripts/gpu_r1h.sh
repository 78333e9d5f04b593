export PYTHONUNBUFFERED=1
timeout 200 python -m pytest tests/test_exec_gpu.py tests/test_runtime_gpu.py -x -q -m gpu 2>&1 | tail -3
timeout 120 python scripts/kb_probe.py 2>&1 | grep -E "==|steady|cta0 issue"
FTB_PAIR=0 timeout 200 python scripts/gemm_probe.py 2>&1 | grep -v cuBLAS | tail -6
FTB_PAIR=1 timeout 200 python scripts/gemm_probe.py 2>&1 | grep -v cuBLAS | tail -6
for p in 0 1; do
  for ops in dense bmm all; do
    FTB_PAIR=$p timeout 120 python bench.py --steps 20 --warmup 5 --ops $ops --no-cpu --per-shape 0 --min-warm-s 0.3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pair=$p $ops', round(d['ms_per_step'],4), 'ms', round(d['value'],1), 'TF/s frac', round(d['roofline']['frac'],3))" 2>&1 | tail -2
  done
done
