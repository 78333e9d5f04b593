SHAPES="dense 16 4096 4096;dense 160 768 3072" CL=1 NL=6 python scripts/chain_trace.py 2>&1 | grep -E "reducing|cluster clk|us/launch|L2:"
S="dense 1 4096 4096;dense 16 4096 4096;dense 64 4096 4096;dense 127 4096 4096;dense 256 4096 4096;dense 160 768 3072;dense 352 768 3072;dense 608 768 3072;dense 768 768 3072;dense 1024 768 3072;dense 1536 768 3072"
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_prev.so python scripts/chain_time.py 2>&1 | sed 's/cfg {.*}//'
SHAPES="$S" python scripts/chain_time.py 2>&1 | sed 's/cfg {.*}//'
