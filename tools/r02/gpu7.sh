#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02g_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo "rc=$?" >> gpurun_out/r02g_bench.err
timeout 900 python bench.py --config reddit-gcn56-eas --steps 5 --warmup 3 --no-hbm-pass > gpurun_out/r02g_gcn56.json 2> gpurun_out/r02g_gcn56.err; echo "rc=$?" >> gpurun_out/r02g_gcn56.err
timeout 600 python bench.py --config products-gcn --steps 10 --warmup 3 > gpurun_out/r02g_products.json 2> gpurun_out/r02g_products.err; echo "rc=$?" >> gpurun_out/r02g_products.err
tail -2 gpurun_out/r02g_smoke.log; for f in bench gcn56 products; do tail -3 gpurun_out/r02g_$f.err; python -c "
import json,sys
d=json.loads(open('gpurun_out/r02g_$f.json').read().strip().splitlines()[-1])
r=d['roofline']
print('$f', d['value'], 'e2e', d['e2e'] and d['e2e']['value'], 'loss1', d['loss_epoch1'], 'after', d['loss_after'], 'parity', d['parity'], 'frac', r['bound'], r['frac'], 'share', r['share_of_step'], 'graph', d['cuda_graph'], 'launches', d['gpu_launches'])
print(json.dumps(r.get('hbm_regime'))[:400])
"; done
