S="dense 128 256 64;dense 608 768 768;dense 160 2304 768;dense 768 3072 768;dense 1472 2304 768;dense 352 2304 768;dense 3808 768 768"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2ad.txt 2>&1
SHAPES="$S" FTB_DIRECT_STORE=1 python scripts/chain_time.py >> gpurun_out/r2ad.txt 2>&1
cat gpurun_out/r2ad.txt | cut -c 1-62,180-230
FTB_DIRECT_STORE=1 timeout 900 python -m pytest tests/test_exec_gpu.py tests/test_runtime_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
