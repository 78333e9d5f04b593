timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2ba_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r2ba_pytest.txt
S="dense 128 256 64;dense 160 768 768;dense 352 768 768;dense 608 768 768;dense 1024 768 768;dense 160 2304 768;dense 352 2304 768;dense 160 3072 768;dense 160 768 3072;dense 768 768 3072"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2ba.txt 2>&1
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2ba_bench.json 2> gpurun_out/r2ba_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2ba_bench.json'));print(d['value'],d['shape_set_mean_roofline_frac'],d['shape_set_p10_roofline_frac'],d['shape_set_frac_by_kind'],d['grouped_step'],d['e2e']['value'])"
cat gpurun_out/r2ba.txt
