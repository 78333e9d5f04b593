S="dense 1024 768 3072;dense 160 768 3072;dense 256 4096 4096"
SHAPES="$S" FTB_TMA_STORE=0 python scripts/chain_time.py > gpurun_out/r2m_ab.txt 2>&1
SHAPES="$S" FTB_L2_PREFETCH=0 python scripts/chain_time.py >> gpurun_out/r2m_ab.txt 2>&1
SHAPES="$S" FTB_TMA_STORE=0 FTB_LIB=paper_2407_21418_b200/libftb_base.so python scripts/chain_time.py >> gpurun_out/r2m_ab.txt 2>&1
CL=1 SHAPES="dense 160 768 3072" NL=4 python scripts/chain_trace.py >> gpurun_out/r2m_ab.txt 2>&1
CL=1 FTB_TMA_STORE=0 SHAPES="dense 160 768 3072" NL=4 python scripts/chain_trace.py >> gpurun_out/r2m_ab.txt 2>&1
cat gpurun_out/r2m_ab.txt | cut -c 1-250
