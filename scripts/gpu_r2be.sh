S="bmm 384 23 23 64 nk;bmm 384 15 15 64 nk;bmm 384 31 31 64 nk;bmm 384 39 39 64 nk;bmm 384 45 45 64 nk;bmm 384 23 64 23 kn;bmm 384 45 64 45 kn"
SHAPES="$S" python scripts/chain_time.py > gpurun_out/r2be.txt 2>&1
SHAPES="$S" FTB_TMA_TAIL_MIN=8 python scripts/chain_time.py >> gpurun_out/r2be.txt 2>&1
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2be_bench.json 2> gpurun_out/r2be_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2be_bench.json'));print(d['value'],d['shape_set_mean_roofline_frac'],d['shape_set_p10_roofline_frac'],d['shape_set_frac_by_kind'],d['grouped_step']['ms_per_step'],d['e2e']['value'])"
cat gpurun_out/r2be.txt
