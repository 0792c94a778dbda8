#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2; do
for cfg in "GDX_P24_UN=4 GDX_P24_MINB=4" "GDX_P24_UN=2 GDX_P24_MINB=6" "GDX_P24_UN=2 GDX_P24_MINB=4" "GDX_P24_UN=2 GDX_P24_MINB=8"; do
  env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --no-hbm-pass --no-e2e --no-cpu-baseline > gpurun_out/pt.json 2> gpurun_out/pt.err
  python -c "import json; d=json.loads(open('gpurun_out/pt.json').read().strip().splitlines()[-1]); print('$cfg', d['ms_per_step'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pt.err
done; done
