CL=1 SHAPES="dense 1024 768 3072;dense 160 768 3072" NL=4 python scripts/chain_trace.py > gpurun_out/r2k_trace.txt 2>&1
CL=1 FTB_SPLIT_WIDE_CLUSTER=1 SHAPES="dense 608 768 768" NL=4 python scripts/chain_trace.py >> gpurun_out/r2k_trace.txt 2>&1
cat gpurun_out/r2k_trace.txt
