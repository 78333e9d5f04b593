python scripts/chain_trace.py > gpurun_out/r2c_chain_trace.txt 2>&1; echo rc=$?
FTB_PDL=0 SHAPES="bmm 384 5 5 64 nk;dense 608 768 768" python scripts/chain_trace.py > gpurun_out/r2c_chain_trace_nopdl.txt 2>&1
cat gpurun_out/r2c_chain_trace.txt gpurun_out/r2c_chain_trace_nopdl.txt
