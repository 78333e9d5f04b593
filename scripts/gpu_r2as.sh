# end-of-CTA wait on store reads only vs full completion; pair-kernel role profile
S="dense 128 256 64;dense 608 768 768;dense 160 2304 768;dense 1472 2304 768;dense 4096 3072 768;dense 4096 768 3072;bmm 384 5 5 64 nk;bmm 384 64 64 64 nk"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2as.txt 2>&1
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_endread.so python scripts/chain_time.py >> gpurun_out/r2as.txt 2>&1
SHAPES="$S" python scripts/chain_time.py >> gpurun_out/r2as.txt 2>&1
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_endread.so python scripts/chain_time.py >> gpurun_out/r2as.txt 2>&1
SHAPES="dense 4096 3072 768;dense 1536 3072 768;dense 8192 8192 8192" FTB_PAIR=1 python scripts/prof_chain.py >> gpurun_out/r2as.txt 2>&1
SHAPES="dense 4096 3072 768;dense 4096 768 3072;dense 8192 8192 8192" FTB_LIB=paper_2407_21418_b200/libftb_nullepi.so python scripts/chain_time.py >> gpurun_out/r2as.txt 2>&1
SHAPES="dense 4096 3072 768;dense 4096 768 3072;dense 8192 8192 8192" FTB_PAIR=1 FTB_LIB=paper_2407_21418_b200/libftb_nullepi.so python scripts/chain_time.py >> gpurun_out/r2as.txt 2>&1
cat gpurun_out/r2as.txt
