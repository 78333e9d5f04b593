# A/B of two trees on the same box: bash scripts/ab_bench.sh DIR_A DIR_B [ops...]
A=$1; B=$2; shift 2
OPS=${@:-all}
for r in 1 2; do for d in $A $B; do for ops in $OPS; do
  (cd $d && timeout 200 python bench.py --steps 30 --warmup 5 --no-cpu --per-shape 0 --min-warm-s 0.5 --ops $ops 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', '$ops', round(d['ms_per_step'],4), 'ms', round(d['value'],1), 'TF/s', d['clocks']['sm_mhz'])")
done; done; done
