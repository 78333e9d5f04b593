timeout 900 python -m pytest tests -m gpu -x -q -k "split or cluster or c3 or fuzz" > gpurun_out/r2bf_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r2bf_pytest.txt
cp paper_2407_21418_b200/libftb.so /tmp/libftb_new.so
S="dense 1 4096 4096;dense 16 4096 4096;dense 64 4096 4096;dense 127 4096 4096;dense 256 4096 4096;dense 160 768 3072;dense 352 768 3072;dense 608 768 3072;dense 768 768 3072;dense 1024 768 3072;dense 1536 768 3072"
SHAPES="$S" FTB_LIB=paper_2407_21418_b200/libftb_prev.so python scripts/chain_time.py > gpurun_out/r2bf.txt 2>&1
SHAPES="$S" python scripts/chain_time.py >> gpurun_out/r2bf.txt 2>&1
cat gpurun_out/r2bf.txt
