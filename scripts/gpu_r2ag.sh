CL=1 SHAPES="dense 160 768 3072;dense 16 4096 4096;dense 1024 768 3072" NL=4 python scripts/chain_trace.py 2>&1 | grep -E "us/launch|cluster clk" | cut -c 1-200
