# A/B of prebuilt libftb.so variants in this tree: bash scripts/ab_libs.sh LIB_A LIB_B ...
# (each copied over paper_2407_21418_b200/libftb.so in turn; step + per-shape mean)
orig=$(mktemp); cp paper_2407_21418_b200/libftb.so $orig
for r in 1 2; do for L in "$@"; do
  src=$L; [ "$(realpath $L)" = "$(realpath paper_2407_21418_b200/libftb.so)" ] && src=$orig  # the live lib: its saved copy
  cp $src paper_2407_21418_b200/libftb.so
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --per-shape-rows --min-warm-s 0.5 2>&1 | tail -1 | python -c "
import json,sys,collections
d=json.loads(sys.stdin.read()); g=collections.defaultdict(list)
for x in d['per_shape']: g[x['name']].append(x['frac'])
print('$L', round(d['ms_per_step'],4), 'ms', d['clocks']['sm_mhz'], 'MHz mean', round(d['shape_set_mean_roofline_frac'],4), {k: round(sum(v)/len(v),3) for k,v in g.items()})"
done; done
cp $orig paper_2407_21418_b200/libftb.so
