timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -3
FTB_PROFILE_CREATE=1 python scripts/prof_create.py 2>&1 | tail -4
timeout 1500 python bench.py --steps 5 --warmup 3 --c4-shapes 0 --no-cpu > gpurun_out/r2s_bench.json 2> gpurun_out/r2s_bench.err; echo bench_rc=$?
tail -5 gpurun_out/r2s_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2s_bench.json').read().strip().split('\n')[-1]); print(json.dumps(d['e2e_dynamic'])); print(d['value'], d['shape_set_mean_roofline_frac'], d['e2e']['value'], d['grouped_step']['ms_per_step'])"
