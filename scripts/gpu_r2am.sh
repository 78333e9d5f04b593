FTB_PAIR=1 SHAPES="dense 4096 3072 768;dense 4096 4096 4096" python scripts/prof_chain.py 2>&1 | tail -8
S="dense 4096 3072 768;dense 3808 2304 768;dense 4096 4096 4096;dense 8192 4096 4096"
SHAPES="$S" python scripts/chain_time.py 2>&1 | cut -c 1-62
SHAPES="$S" FTB_PAIR=1 python scripts/chain_time.py 2>&1 | cut -c 1-62
FTB_PAIR=1 timeout 600 python -m pytest tests/test_exec_gpu.py -x -q -m gpu -p no:cacheprovider -k "pair" 2>&1 | tail -2
