export PYTHONUNBUFFERED=1
FTB_PAIR=0 timeout 200 python scripts/gemm_probe.py 2>&1 | tail -12
FTB_PAIR=1 timeout 200 python scripts/gemm_probe.py 2>&1 | tail -12
timeout 200 python scripts/trace_probe.py 2>&1 | tail -40
