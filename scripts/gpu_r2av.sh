# 64-column split by default: GPU tests, then the default bench command
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2av_pytest.txt 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r2av_pytest.txt
t0=$(date +%s.%N); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2av_bench.json 2> gpurun_out/r2av_bench.err; echo rc=$? wall=$(echo "$(date +%s.%N) - $t0" | bc)
tail -2 gpurun_out/r2av_bench.err
python -c "import json;d=json.load(open('gpurun_out/r2av_bench.json'));print(d['value'],d['shape_set_mean_roofline_frac'],d['shape_set_p10_roofline_frac'],d['shape_set_frac_by_kind'],d['grouped_step'].get('ms'),d['e2e']['value'])"
