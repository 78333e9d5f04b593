KB=1 FTB_LIB=paper_2407_21418_b200/libftb_tracepre.so SHAPES="dense 608 768 768;dense 128 256 64;bmm 384 5 5 64 nk" NL=4 FTB_SPLIT_WIDE_CLUSTER=0 python scripts/chain_trace.py > gpurun_out/r2i_trace.txt 2>&1
cat gpurun_out/r2i_trace.txt
