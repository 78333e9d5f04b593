# epilogue share of the launch: release vs epilogue-without-stores vs no epilogue at all; role profile of big shapes
S="dense 128 256 64;dense 608 768 768;dense 160 2304 768;dense 1472 2304 768;dense 1536 3072 768;dense 4096 3072 768;dense 4096 768 3072;bmm 384 5 5 64 nk;bmm 384 64 64 64 nk;bmm 384 100 100 64 nk"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2ar.txt 2>&1
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_nostore.so python scripts/chain_time.py >> gpurun_out/r2ar.txt 2>&1
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_nullepi.so python scripts/chain_time.py >> gpurun_out/r2ar.txt 2>&1
SHAPES="dense 4096 3072 768;dense 4096 768 3072;dense 1536 3072 768;dense 8192 8192 8192" python scripts/prof_chain.py >> gpurun_out/r2ar.txt 2>&1
cat gpurun_out/r2ar.txt
