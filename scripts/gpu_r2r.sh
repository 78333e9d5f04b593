timeout 1500 python bench.py --steps 5 --warmup 3 --c4-shapes 0 --no-cpu > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; echo bench_rc=$?
tail -5 gpurun_out/r2r_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2r_bench.json').read().strip().split('\n')[-1]); print(json.dumps(d['e2e_dynamic'])); print(d['value'], d['shape_set_mean_roofline_frac'], d['e2e'])"
