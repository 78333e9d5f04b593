S="dense 608 768 768;dense 160 2304 768;dense 1024 768 3072;dense 160 768 3072;dense 768 3072 768;dense 64 4096 4096;dense 256 4096 4096"
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_base.so python scripts/chain_time.py > gpurun_out/r2l_ab.txt 2>&1
SHAPES="$S" python scripts/chain_time.py >> gpurun_out/r2l_ab.txt 2>&1
SHAPES="$S" FTB_SPLIT_WIDE_CLUSTER=1 python scripts/chain_time.py >> gpurun_out/r2l_ab.txt 2>&1
SHAPES="$S" FTB_SPLIT_WIDE_CLUSTER=1 FTB_SPLIT_CL_MINKB=2 python scripts/chain_time.py >> gpurun_out/r2l_ab.txt 2>&1
cat gpurun_out/r2l_ab.txt | awk '{print $1,$2,$3,$4,$5,$6,$8,$10,$12, $NF}'
timeout 900 python -m pytest tests/test_exec_gpu.py -x -q -m gpu -p no:cacheprovider -k "split or graph or eight" 2>&1 | tail -5
FTB_SPLIT_WIDE_CLUSTER=1 timeout 900 python -m pytest tests/test_exec_gpu.py tests/test_fuzz_gpu.py tests/test_runtime_gpu.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -5
