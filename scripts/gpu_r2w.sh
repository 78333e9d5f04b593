CL=1 KB=1 SHAPES="dense 16 4096 4096;dense 256 4096 4096" NL=4 python scripts/chain_trace.py 2>&1 | cut -c 1-250
