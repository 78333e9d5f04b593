export PYTHONUNBUFFERED=1
FTB_PAIR=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:ftb_tc_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_single python scripts/gemm_one.py > gpurun_out/ncu_gs.log 2>&1; tail -2 gpurun_out/ncu_gs.log
FTB_PAIR=1 TI=256 timeout 300 ncu --set full --clock-control none --import-source on -k regex:ftb_tc2_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_pair python scripts/gemm_one.py > gpurun_out/ncu_gp.log 2>&1; tail -2 gpurun_out/ncu_gp.log
