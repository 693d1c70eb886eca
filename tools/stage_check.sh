# pageable staging: parity tests and the bench's pageable / drop-in e2e legs
set -x
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "pageable or host" 2>&1 | tail -3
OZK_BENCH_NO_CPU=1 python bench.py --steps 3 --warmup 3 > gpurun_out/stage_bench.json 2> gpurun_out/stage_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/stage_bench.json').read().strip().splitlines()[-1])
print(d['value'], json.dumps(d['e2e']), json.dumps(d.get('e2e_pageable')), json.dumps(d.get('e2e_dropin')))"
