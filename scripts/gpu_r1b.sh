for ops in dense bmm; do
  timeout 300 python bench.py --steps 20 --warmup 5 --ops $ops --no-cpu --per-shape 0 --min-warm-s 0.3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$ops', d['ms_per_step'], d['value'], d['work_items'], d['roofline'])"
done
timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu --per-shape-rows --min-warm-s 0.3 > gpurun_out/bench_ps.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_ps.json').read().strip().splitlines()[-1])
print('mean frac', d['shape_set_mean_roofline_frac'], 'mean tflops', d['shape_set_mean_tflops'])
for r in d['per_shape'][:48]: print(r['name'], r['b'], r['M'], r['N'], r['K'], round(r['us'],2), round(r['tflops'],1), round(r['frac'],3), r['bound'])
"
