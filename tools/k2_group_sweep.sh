# K2 raster group size sweep: the bench step on one box
# (alternating configurations), then DRAM bytes per K2 launch (ncu).
one() { env OZK_K2_GROUP=$1 OZK_BENCH_NO_CPU=1 python bench.py --no-extra --no-e2e --steps 10 --warmup 3 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print(json.dumps({'G': $1, 'value': round(d['value'],2), 'sm_mhz': d['clocks']['sm_mhz'], 'k2_ms': round(r['k2_ms'],3)}))"; }
for rep in 1 2; do for g in ${KGROUPS:-4 6 8 12 16}; do one $g; done; done
for g in ${KGROUPS:-4 6 8 12 16}; do
  echo "G=$g"
  OZK_K2_GROUP=$g OZK_BENCH_NO_CPU=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:residue_gemm -s 4 -c 1 --csv python bench.py --no-extra --no-e2e --steps 2 --warmup 3 2>/dev/null | grep -E "dram__bytes|gpu__time|cycles_elapsed|hit_rate" | python -c "
import csv,sys
for r in csv.reader(sys.stdin): print('  ', r[-3], r[-2], r[-1])"
done
