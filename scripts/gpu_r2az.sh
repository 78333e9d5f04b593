S="dense 128 256 64;dense 160 768 768;dense 352 768 768;dense 608 768 768;dense 1024 768 768;dense 160 2304 768;dense 352 2304 768;dense 160 3072 768;dense 160 768 3072;dense 768 768 3072"
for V in "FTB_COLSPLIT_MIN=64" "FTB_COLSPLIT_MIN=32" "FTB_COLSPLIT_MIN=64" "FTB_COLSPLIT_MIN=32"; do env $V SHAPES="$S" python scripts/chain_time.py >> gpurun_out/r2az.txt 2>&1; done
