SHAPES="dense 608 768 768;dense 768 3072 768" NL=4 python scripts/chain_trace.py > gpurun_out/r2h_trace.txt 2>&1
SHAPES="dense 608 768 768;dense 768 3072 768" NL=4 FTB_SPLIT_WIDE_CLUSTER=0 python scripts/chain_trace.py >> gpurun_out/r2h_trace.txt 2>&1
cat gpurun_out/r2h_trace.txt
