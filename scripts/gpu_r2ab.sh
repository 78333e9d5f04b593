S="dense 128 256 64;dense 608 768 768;dense 160 2304 768;dense 768 3072 768;dense 1472 2304 768;bmm 384 5 5 64 nk;bmm 384 46 46 64 nk;bmm 384 46 64 46 kn;bmm 384 64 64 64 nk"
SHAPES="$S" FTB_EPI8_SPLIT=0 python scripts/chain_time.py > gpurun_out/r2ab.txt 2>&1
SHAPES="$S" python scripts/chain_time.py >> gpurun_out/r2ab.txt 2>&1
cat gpurun_out/r2ab.txt | cut -c 1-62,180-230
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
