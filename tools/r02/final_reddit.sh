#!/bin/bash
# final tree: Reddit bench lines at N=1/2/4 (full contract: e2e with the live floor, parity at N=1)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/fr; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/reddit-sage_n1.json 2> $O/reddit-sage_n1.err
for n in 2 4; do
  timeout 900 $R --nproc-per-node $n --master-port 2981$n bench.py --gpus $n --steps 20 --warmup 5 > $O/reddit-sage_n$n.json 2> $O/reddit-sage_n$n.err
done
for f in $O/*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1], d['n_gpus'], d['value'], 'e2e', d['e2e']['value'], 'floor', d['e2e']['pcie_floor_ms'], 'par', (d.get('parity') or {}).get('abs_diff'), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
