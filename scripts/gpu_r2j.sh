S="dense 128 256 64;dense 608 768 768;dense 160 2304 768;dense 1024 768 3072;dense 3200 768 3072;bmm 384 5 5 64 nk;bmm 384 46 46 64 nk;bmm 384 100 100 64 nk;bmm 384 46 64 46 kn"
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_base.so python scripts/chain_time.py > gpurun_out/r2j_ab.txt 2>&1
SHAPES="$S" FTB_L2_PREFETCH=0 python scripts/chain_time.py >> gpurun_out/r2j_ab.txt 2>&1
SHAPES="$S" python scripts/chain_time.py >> gpurun_out/r2j_ab.txt 2>&1
cat gpurun_out/r2j_ab.txt
