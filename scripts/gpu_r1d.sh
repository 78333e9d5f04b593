export PYTHONUNBUFFERED=1
timeout 180 python -m pytest tests/test_exec_gpu.py -x -q -m gpu 2>&1 | tail -4
for p in 0 1; do
  for ops in dense all; do
    FTB_PAIR=$p timeout 120 python bench.py --steps 20 --warmup 5 --ops $ops --no-cpu --per-shape 0 --min-warm-s 0.3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pair=$p $ops', round(d['ms_per_step'],4), 'ms', round(d['value'],1), 'TF/s frac', round(d['roofline']['frac'],3))" 2>&1 | tail -2
  done
done
FTB_PAIR=1 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu --per-shape-rows --min-warm-s 0.3 > gpurun_out/bench_v3.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_v3.json').read().strip().splitlines()[-1])
print('step ms', d['ms_per_step'], 'TF/s', d['value'], 'frac', d['roofline']['frac'], 'mean frac', d['shape_set_mean_roofline_frac'])
for r in d['per_shape'][:24]: print(r['name'], r['b'], r['M'], r['N'], r['K'], round(r['us'],2), round(r['tflops'],1), round(r['frac'],3), r['bound'])
" 2>&1 | tail -30
