t0=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2bm_bench.json 2> gpurun_out/r2bm_bench.err; echo rc=$? wall=$(( $(date +%s) - t0 ))s
tail -2 gpurun_out/r2bm_bench.err
t0=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2bm_ref.json 2> gpurun_out/r2bm_ref.err; echo rc=$? wall=$(( $(date +%s) - t0 ))s
tail -2 gpurun_out/r2bm_ref.err; cat gpurun_out/r2bm_ref.json | cut -c1-400
python -c "import json;d=json.load(open('gpurun_out/r2bm_bench.json'));print(d['value'],d['shape_set_mean_roofline_frac'],d['shape_set_p10_roofline_frac'],d['shape_set_frac_by_kind'],d['grouped_step']['ms_per_step'],d['grouped_step']['roofline'],d['e2e'],d['roofline'],d['clocks'],d['c4_sweep']['tflops'],d['c4_sweep']['roofline_frac'],d.get('e2e_dynamic',{}) and {k:v for k,v in d['e2e_dynamic'].items() if k!='per_step'})"
