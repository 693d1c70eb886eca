# One-pass K1 A/B on one box: the bench step with OZK_K1_FUSED = 1 (column
# kernel, the default), 0 (two-kernel path) and 3 (column + row kernel),
# alternating, then the ncu launch list of each setting.
summ() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);r=d['roofline'];print(json.dumps({'fused': sys.argv[2], 'value': round(d['value'],2), 'k1_ms': round(r['k1_ms'],3), 'k2_ms': round(r['k2_ms'],3), 'k3_ms': round(r['k3_ms'],3), 'sm_mhz': d['clocks']['sm_mhz']}))" $1 "$2"; }
mkdir -p gpurun_out
for rep in 1 2; do for f in ${MASKS:-1 0 3}; do
  OZK_K1_FUSED=$f OZK_BENCH_NO_CPU=1 python bench.py --no-extra --no-e2e --steps 10 --warmup 3 > gpurun_out/_ab.json 2>/dev/null; summ gpurun_out/_ab.json $f
done; done
for f in ${MASKS:-1 0 3}; do
  echo "launches OZK_K1_FUSED=$f"
  OZK_K1_FUSED=$f OZK_BENCH_NO_CPU=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/_ab_launches_$f.csv python bench.py --steps 1 --warmup 1 --no-extra --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py launches gpurun_out/_ab_launches_$f.csv | grep -v "at::" | head -8
done
