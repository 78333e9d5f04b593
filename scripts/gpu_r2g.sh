S="dense 608 768 768;dense 1024 768 3072;dense 160 2304 768;dense 768 3072 768;dense 1472 2304 768;dense 3200 768 3072;dense 160 768 3072"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2g_chain_time.txt 2>&1
SHAPES="$S" FTB_SPLIT_WIDE_CLUSTER=0 python scripts/chain_time.py >> gpurun_out/r2g_chain_time.txt 2>&1
SHAPES="$S" FTB_SPLIT_CL_MINKB=2 python scripts/chain_time.py >> gpurun_out/r2g_chain_time.txt 2>&1
cat gpurun_out/r2g_chain_time.txt
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -5
