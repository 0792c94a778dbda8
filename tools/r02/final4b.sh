#!/bin/bash
# 4-GPU box, final round-2 tree: bench lines at N=1/2/4 for every config, the reference
# arm, and the multi-GPU parity test (dist_check at N=4 incl. the packed-24 trainer).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/final2; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_multi_gpu.py -q -m gpu > $O/multi_gpu_pytest.log 2>&1; echo "multi-gpu pytest rc=$? $(tail -1 $O/multi_gpu_pytest.log)"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/reddit-sage_n1.json 2> $O/reddit-sage_n1.err
for n in 2 4; do
  timeout 900 $R --nproc-per-node $n --master-port 2959$n bench.py --gpus $n --steps 20 --warmup 5 > $O/reddit-sage_n$n.json 2> $O/reddit-sage_n$n.err
done
for cfg in products-gcn reddit-gcn56-eas; do
  steps=20; [ $cfg = reddit-gcn56-eas ] && steps=5
  timeout 900 python bench.py --config $cfg --steps $steps --warmup 5 > $O/${cfg}_n1.json 2> $O/${cfg}_n1.err
  for n in 2 4; do
    timeout 900 $R --nproc-per-node $n --master-port 2958$n bench.py --gpus $n --config $cfg --steps $steps --warmup 5 > $O/${cfg}_n$n.json 2> $O/${cfg}_n$n.err
  done
done
timeout 2000 $R --nproc-per-node 4 --master-port 29577 bench.py --gpus 4 --config papers-cobatch --steps 2 --warmup 3 > $O/papers-cobatch_n4.json 2> $O/papers-cobatch_n4.err
timeout 2000 python bench.py --config papers-cobatch --steps 2 --warmup 3 > $O/papers-cobatch_n1.json 2> $O/papers-cobatch_n1.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/reference_n1.json 2> $O/reference_n1.err
for f in $O/*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1])
    r=d.get('roofline') or {}
    print('$f'.split('/')[-1], d.get('n_gpus'), d.get('value'), 'e2e', (d.get('e2e') or {}).get('value'), 'par', (d.get('parity') or {}).get('abs_diff'), 'frac', r.get('frac'), 'gather', (r.get('gather_ceiling') or {}).get('frac'), 'clk', (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))
except Exception as e: print('$f', 'FAIL', e)
"; done
