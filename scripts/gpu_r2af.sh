t0=$(date +%s.%N); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2af_bench.json 2> gpurun_out/r2af_bench.err; echo rc=$? wall=$(echo "$(date +%s.%N) - $t0" | bc)
tail -2 gpurun_out/r2af_bench.err
t0=$(date +%s.%N); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2af_ref.json 2> gpurun_out/r2af_ref.err; echo rc=$? wall=$(echo "$(date +%s.%N) - $t0" | bc)
tail -2 gpurun_out/r2af_ref.err; cat gpurun_out/r2af_ref.json
