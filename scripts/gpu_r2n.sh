S="dense 1024 768 3072;dense 160 768 3072;dense 256 4096 4096;dense 608 768 768;dense 768 3072 768"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2n_ab.txt 2>&1
SHAPES="$S" FTB_SPLIT_WIDE_CLUSTER=1 python scripts/chain_time.py >> gpurun_out/r2n_ab.txt 2>&1
CL=1 SHAPES="dense 160 768 3072" NL=4 python scripts/chain_trace.py >> gpurun_out/r2n_ab.txt 2>&1
cat gpurun_out/r2n_ab.txt | cut -c 1-200
