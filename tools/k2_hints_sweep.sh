# Recipe of profiles/r01_k2_hints_sweep.md (run on the GPU box: bash tools/k2_hints_sweep.sh).
# Hint bit 2 (streaming U stores) has since been removed; 4/5/13 now equal 0/1/9.
export SWEEP_VARIANTS='[{"OZK_K2_SYNC":"1","OZK_K2_GROUP":"8","OZK_K2_HINTS":"0"},{"OZK_K2_SYNC":"1","OZK_K2_GROUP":"8","OZK_K2_HINTS":"1"},{"OZK_K2_SYNC":"1","OZK_K2_GROUP":"8","OZK_K2_HINTS":"4"},{"OZK_K2_SYNC":"1","OZK_K2_GROUP":"8","OZK_K2_HINTS":"5"},{"OZK_K2_SYNC":"1","OZK_K2_GROUP":"8","OZK_K2_HINTS":"9"},{"OZK_K2_SYNC":"1","OZK_K2_GROUP":"8","OZK_K2_HINTS":"13"},{"OZK_K2_SYNC":"1","OZK_K2_GROUP":"16","OZK_K2_HINTS":"13"},{"OZK_K2_SYNC":"1","OZK_K2_GROUP":"6","OZK_K2_HINTS":"0"}]'
SWEEP_REPS=3 python tools/k2_sweep.py > gpurun_out/sweep_time.jsonl 2>&1
SWEEP_REPS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none --csv python tools/k2_sweep.py > gpurun_out/sweep_ncu.csv 2>&1
