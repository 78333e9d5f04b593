S="dense 128 256 64;dense 608 768 768;dense 1024 768 3072;dense 16 4096 4096;bmm 384 5 5 64 nk;bmm 384 46 46 64 nk;bmm 384 100 100 64 nk;bmm 384 46 64 46 kn"
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_base.so python scripts/chain_time.py > gpurun_out/r2z_ab.txt 2>&1
SHAPES="$S" python scripts/chain_time.py >> gpurun_out/r2z_ab.txt 2>&1
cat gpurun_out/r2z_ab.txt | awk '{print $1,$2,$3,$4,$5,$6,$NF}'
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
