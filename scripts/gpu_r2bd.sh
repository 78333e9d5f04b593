timeout 600 python -m pytest tests/test_exec_gpu.py -x -q -k "tail or bulk_row or padding" > gpurun_out/r2bd_pytest.txt 2>&1; echo tail_rc=$?; tail -3 gpurun_out/r2bd_pytest.txt
timeout 1500 python -m pytest tests -m gpu -x -q >> gpurun_out/r2bd_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r2bd_pytest.txt
S="bmm 384 96 96 64 nk;bmm 384 95 95 64 nk;bmm 384 97 97 64 nk;bmm 384 63 63 64 nk;bmm 384 121 121 64 nk;bmm 384 23 23 64 nk;bmm 384 15 15 64 nk;bmm 384 5 5 64 nk;bmm 1024 257 257 64 nk;bmm 1024 255 255 64 nk"
SHAPES="$S;bmm 384 50 50 64 nk;bmm 384 57 57 64 nk;bmm 384 60 60 64 nk" FTB_TMA_TAIL=0 python scripts/chain_time.py > gpurun_out/r2bd.txt 2>&1
SHAPES="$S;bmm 384 50 50 64 nk;bmm 384 57 57 64 nk;bmm 384 60 60 64 nk" python scripts/chain_time.py >> gpurun_out/r2bd.txt 2>&1
cat gpurun_out/r2bd.txt
