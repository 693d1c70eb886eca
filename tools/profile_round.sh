#!/bin/bash
# One-GPU evidence for profiles/: the bench line, the ncu launch list of one
# bench step, and one `ncu --set full` capture of each pipeline kernel.
# usage (on the GPU box): bash tools/profile_round.sh <tag>
set -x
tag=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
OZK_BENCH_NO_CPU=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 1 --no-extra --no-e2e > gpurun_out/launches_$tag.log 2>&1
OZK_BENCH_NO_CPU=1 ncu --set full --clock-control none --import-source on \
  -k "regex:residue_gemm|planes_kernel|reconstruct|row_stats|col_stats|fused_kernel" -c 5 \
  -o gpurun_out/full_$tag python bench.py --steps 1 --warmup 0 --no-extra --no-e2e > gpurun_out/full_$tag.log 2>&1
ls -la gpurun_out
