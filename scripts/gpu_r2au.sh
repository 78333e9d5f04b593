# narrower column split (64-column pieces) for one-wave tables: store tail vs MMA-N floor
S="dense 160 768 768;dense 608 768 768;dense 1024 768 768;dense 160 2304 768;dense 352 2304 768;dense 160 3072 768;dense 608 3072 768;dense 160 768 3072;dense 352 768 3072;dense 768 768 3072;dense 128 256 64"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2au.txt 2>&1
SHAPES="$S" FTB_COLSPLIT_MIN=64 python scripts/chain_time.py >> gpurun_out/r2au.txt 2>&1
SHAPES="$S" python scripts/chain_time.py >> gpurun_out/r2au.txt 2>&1
SHAPES="$S" FTB_COLSPLIT_MIN=64 python scripts/chain_time.py >> gpurun_out/r2au.txt 2>&1
cat gpurun_out/r2au.txt
