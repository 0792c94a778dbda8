#!/bin/bash
# packed-24 kernel occupancy A/B (MINB 5 = 48-register cap, 40 warps/SM) + the fixed gather probe
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2; do
for cfg in "GDX_P24_MINB=4" "GDX_P24_MINB=5" "GDX_P24_UN=2 GDX_P24_MINB=5"; do
  env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --no-hbm-pass --no-e2e --no-cpu-baseline > gpurun_out/m5.json 2> gpurun_out/m5.err
  python -c "import json; d=json.loads(open('gpurun_out/m5.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$cfg', d['ms_per_step'], r['avg_launch_ms'], d['clocks']['sm_mhz'], 'l2', r['l2_probe_gbs'], 'gather', r['gather_ceiling']['peak'], r['gather_ceiling']['frac'])" || tail -3 gpurun_out/m5.err
done; done
