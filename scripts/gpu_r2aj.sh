python scripts/c0_time.py 2>&1 | tail -8
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "ffma or c0 or fp32" 2>&1 | tail -3
