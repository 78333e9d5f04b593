# Run mcast_bench MODE 0/1 alternately, each ~2.5 s, with SM clock / power sampling (median of the in-run samples)
cd "$(dirname "$0")"
for r in 1 2; do for m in ${MODES:-0 1}; do
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/clk_$m.txt &
  SPID=$!
  sleep 0.3
  MODE=$m SECS=2.5 timeout 60 ./mcast_bench
  kill $SPID 2>/dev/null; wait $SPID 2>/dev/null
  python3 - "$m" <<'PY'
import statistics, sys
m = sys.argv[1]
v = [l.split(",") for l in open(f"/tmp/clk_{m}.txt") if l.strip()]
c = [int(x[0]) for x in v if x[0].strip().isdigit()]
p = [float(x[1]) for x in v if len(x) > 1 and x[1].strip().replace(".", "").isdigit()]
c, p = c[4:-2] or c, p[4:-2] or p
print(f"   MODE={m}: SM MHz median {statistics.median(c) if c else None}, power W median {statistics.median(p) if p else None}, samples {len(c)}")
PY
done; done
