# one ncu --set full capture of each K3 variant, isolated (tools/k3_time.py, N = 14)
for v in "OZK_K3_TILE=1" "OZK_K3_CW=4"; do
  tag=$(echo $v | tr '=' '_')
  env $v K3_MODS=14 K3_REPS=2 ncu --set full --clock-control none --import-source on -k regex:reconstruct_tc -s 1 -c 1 \
     -o gpurun_out/k3_$tag python tools/k3_time.py > gpurun_out/k3_$tag.log 2>&1
done
