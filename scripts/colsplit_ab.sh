# A/B of executor switches on the per-shape sweep: VARS="FTB_COLSPLIT=0 FTB_COLSPLIT=1"
for v in ${VARS:-"FTB_COLSPLIT=0" "FTB_COLSPLIT=1"}; do env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --per-shape-rows 2>&1 | tail -1 | python -c "
import json,sys,collections
d=json.loads(sys.stdin.read()); g=collections.defaultdict(list)
for r in d['per_shape']: g[r['name']].append(r['frac'])
print('$v', round(d['ms_per_step'],4), round(d['shape_set_mean_roofline_frac'],4), {k: round(sum(v)/len(v),3) for k,v in g.items()})"; done
