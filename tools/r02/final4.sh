#!/bin/bash
# 4-GPU box: bench lines at N=1 and N=4 for every config, the reference arm (N=1)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 900 python bench.py --steps 20 --warmup 5 > $O/reddit-sage_n1.json 2> $O/reddit-sage_n1.err
for cfg in products-gcn reddit-gcn56-eas; do
  steps=20; [ $cfg = reddit-gcn56-eas ] && steps=5
  timeout 900 python bench.py --config $cfg --steps $steps --warmup 5 > $O/${cfg}_n1.json 2> $O/${cfg}_n1.err
done
for cfg in reddit-sage products-gcn reddit-gcn56-eas; do
  steps=20; [ $cfg = reddit-gcn56-eas ] && steps=5
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29591 bench.py --gpus 4 --config $cfg --steps $steps --warmup 5 > $O/${cfg}_n4.json 2> $O/${cfg}_n4.err
done
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29592 bench.py --gpus 4 --config papers-cobatch --steps 2 --warmup 3 > $O/papers-cobatch_n4.json 2> $O/papers-cobatch_n4.err
timeout 2400 python bench.py --config papers-cobatch --steps 2 --warmup 3 > $O/papers-cobatch_n1.json 2> $O/papers-cobatch_n1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/reference_n1.json 2> $O/reference_n1.err
for f in $O/*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1])
    print('$f'.split('/')[-1], d.get('n_gpus'), d.get('value'), 'e2e', (d.get('e2e') or {}).get('value'), 'par', (d.get('parity') or {}).get('abs_diff'), 'frac', (d.get('roofline') or {}).get('frac'))
except Exception as e: print('$f', 'FAIL', e)
"; done
