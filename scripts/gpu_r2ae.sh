S="dense 4096 3072 768;dense 3808 2304 768;dense 4096 4096 4096;dense 8192 4096 4096;dense 2048 3072 768"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2ae.txt 2>&1
SHAPES="$S" FTB_PAIR=1 python scripts/chain_time.py >> gpurun_out/r2ae.txt 2>&1
cat gpurun_out/r2ae.txt | cut -c 1-62,100-200
