./scripts/micro/launch_floor > gpurun_out/r2e_launch_floor.txt 2>&1
S="dense 128 256 64;dense 608 768 768;bmm 384 5 5 64 nk;bmm 384 100 100 64 nk;dense 160 768 3072"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2e_chain_time.txt 2>&1
SHAPES="$S" FTB_TMA_STORE=0 python scripts/chain_time.py >> gpurun_out/r2e_chain_time.txt 2>&1
SHAPES="$S" FTB_EPI8=0 python scripts/chain_time.py >> gpurun_out/r2e_chain_time.txt 2>&1
SHAPES="$S" FTB_PDL=0 python scripts/chain_time.py >> gpurun_out/r2e_chain_time.txt 2>&1
SHAPES="$S" NL=4 python scripts/chain_time.py >> gpurun_out/r2e_chain_time.txt 2>&1
cat gpurun_out/r2e_launch_floor.txt gpurun_out/r2e_chain_time.txt
