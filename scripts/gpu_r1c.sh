timeout 300 python -m pytest tests/test_exec_gpu.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python scripts/trace_probe.py 2>&1 | tail -60
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --per-shape-rows --min-warm-s 0.3 > gpurun_out/bench_v2.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_v2.json').read().strip().splitlines()[-1])
print('step ms', d['ms_per_step'], 'TF/s', d['value'], 'frac', d['roofline']['frac'], 'mean frac', d['shape_set_mean_roofline_frac'])
for r in d['per_shape'][:24]: print(r['name'], r['b'], r['M'], r['N'], r['K'], round(r['us'],2), round(r['tflops'],1), round(r['frac'],3), r['bound'])
"
