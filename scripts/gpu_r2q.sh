timeout 600 python -m pytest tests/test_runtime_gpu.py -x -q -m gpu -p no:cacheprovider -k "sharded or c1_grouped" 2>&1 | tail -3
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err; echo bench_rc=$?
tail -5 gpurun_out/r2q_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2q_bench.json').read().strip().split('\n')[-1]); print(json.dumps(d['c4_sweep'])); print(d['value'], d['shape_set_mean_roofline_frac'])"
