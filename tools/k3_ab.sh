# K3 A/B on one box: parity, isolated (tools/k3_time.py), right after K2 (tools/insitu_probe.py), one ncu capture
set -x
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "reconstruct or gemm_fp64 or alpha_beta" 2>&1 | tail -2
OZK_K3_REPLAY_ALL=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py -q -x -p no:cacheprovider -k "reconstruct or gemm_fp64 or random" 2>&1 | tail -2
OZK_K3_CW=8 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "reconstruct" 2>&1 | tail -2
for v in "OZK_K3_TILE=1" "OZK_K3_CW=4" "OZK_K3_CW=8" "OZK_K3_STAGES=6"; do echo $v; env $v K3_MODS=8,14,20 python tools/k3_time.py; env $v python tools/insitu_probe.py; done
for v in "OZK_K3_TILE=1" "OZK_K3_CW=4" "OZK_K3_STAGES=6"; do echo $v; env $v OZK_BENCH_NO_CPU=1 python bench.py --no-extra --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print(d['value'], d['clocks'], {k:r[k] for k in r if k.startswith('k')})"; done
K3_MODS=14 K3_REPS=2 ncu --set full --clock-control none --import-source on -k regex:reconstruct_tc -s 1 -c 1 -o gpurun_out/k3_cw4c python tools/k3_time.py > /dev/null 2>&1
