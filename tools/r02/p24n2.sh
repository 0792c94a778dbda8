#!/bin/bash
# N=2: dist_check native modes incl. packed-24, Reddit bench A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${1:-2}
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 \
  tools/dist_check.py --modes native,native-p24,native-eas,sm > gpurun_out/p24n_dist.log 2>&1; echo "dist rc=$?"
grep '^{' gpurun_out/p24n_dist.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ok', d['ok'], {m: v.get('ok') for m, v in d['modes'].items()})"
for v in 1 0; do
  GDX_PACKED24=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 \
    bench.py --gpus $N --steps 20 --warmup 5 --no-hbm-pass > gpurun_out/p24n_reddit_$v.json 2> gpurun_out/p24n_reddit_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/p24n_reddit_$v.json').read().strip().splitlines()[-1]); print('reddit N=$N p24=$v', d['ms_per_step'], d['e2e']['value'])" || tail -5 gpurun_out/p24n_reddit_$v.err
done
