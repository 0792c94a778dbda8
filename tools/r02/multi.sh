#!/bin/bash
# N-GPU session: dist_check sweep, then bench lines for the full-graph configs at N
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${1:-4}
bash tools/r02/dist2.sh $N > gpurun_out/r02_dist_summary_n$N.txt 2>&1
for cfg in reddit-sage products-gcn reddit-gcn56-eas; do
  steps=20; [ $cfg = reddit-gcn56-eas ] && steps=5
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29561 bench.py --gpus $N --config $cfg --steps $steps --warmup 5 \
    > gpurun_out/r02_bench_${cfg}_n$N.json 2> gpurun_out/r02_bench_${cfg}_n$N.err
  echo "rc=$?" >> gpurun_out/r02_bench_${cfg}_n$N.err
done
cat gpurun_out/r02_dist_summary_n$N.txt | tail -16
for cfg in reddit-sage products-gcn reddit-gcn56-eas; do
python -c "
import json
try:
    d=json.loads(open('gpurun_out/r02_bench_${cfg}_n$N.json').read().strip().splitlines()[-1])
    print('$cfg', d['n_gpus'], d['value'], 'e2e', d['e2e'] and d['e2e']['value'], 'loss', d['loss_after'], d['config']['parallelism'][:60])
except Exception as e: print('$cfg fail', e)
"; tail -2 gpurun_out/r02_bench_${cfg}_n$N.err; done
