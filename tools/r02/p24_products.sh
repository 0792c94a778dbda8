#!/bin/bash
# HBM regime: interleaved packed-24 rows on the products-shape GCN epoch (A/B against fp32 rows)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/pp
for i in 1 2; do for v in 0 1; do
  GDX_PACKED24=$v timeout 600 python bench.py --config products-gcn --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/pp/p$v.json 2> gpurun_out/pp/p$v.err
  python -c "import json; d=json.loads(open('gpurun_out/pp/p$v.json').read().strip().splitlines()[-1]); r=d['roofline']; print('p24=$v', d['ms_per_step'], r['avg_launch_ms'], r['achieved'], r['frac'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pp/p$v.err
done; done
GDX_PACKED24=1 timeout 900 python bench.py --config products-gcn --steps 20 --warmup 5 > gpurun_out/pp/p24_full.json 2> gpurun_out/pp/p24_full.err
python -c "import json; d=json.loads(open('gpurun_out/pp/p24_full.json').read().strip().splitlines()[-1]); print('p24 full', d['value'], 'e2e', d['e2e']['value'], 'parity', d['parity'])" || tail -3 gpurun_out/pp/p24_full.err
