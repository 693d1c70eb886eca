# Alternating bench A/B on one box: VARIANTS is a ';'-separated list of
# space-separated env assignments ("" = defaults); REPS rounds of the bench
# step (bench.py --no-extra --no-e2e --steps 10 --warmup 3) per variant,
# one JSON line each with the in-step stage times.
# usage: VARIANTS='OZK_K3_CW=4;OZK_K3_CW=8' REPS=2 bash tools/bench_ab.sh
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for rep in $(seq 1 ${REPS:-2}); do
  for v in "${VS[@]}"; do
    env $v OZK_BENCH_NO_CPU=1 python bench.py --no-extra --no-e2e --steps 10 --warmup 3 ${BENCH_ARGS:-} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(json.dumps({'env': sys.argv[1], 'value': round(d['value'],2), 'k1_ms': round(r['k1_ms'],3), 'k2_ms': round(r['k2_ms'],3), 'k3_ms': round(r['k3_ms'],3), 'sm_mhz': d['clocks']['sm_mhz']}))" "$v"
  done
done
