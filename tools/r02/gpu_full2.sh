#!/bin/bash
# 2-GPU box: the whole -m gpu suite (multi-GPU test included), smoke, N=2 bench lines
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --durations=12 -rf > gpurun_out/r02h_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02h_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02h_smoke.log
for cfg in reddit-sage products-gcn reddit-gcn56-eas; do
  steps=20; [ $cfg = reddit-gcn56-eas ] && steps=5
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29561 bench.py --gpus 2 --config $cfg --steps $steps --warmup 5 \
    > gpurun_out/r02_bench_${cfg}_n2.json 2> gpurun_out/r02_bench_${cfg}_n2.err
  echo "rc=$?" >> gpurun_out/r02_bench_${cfg}_n2.err
done
tail -25 gpurun_out/r02h_pytest_gpu.log; tail -2 gpurun_out/r02h_smoke.log
for cfg in reddit-sage products-gcn reddit-gcn56-eas; do python -c "
import json
d=json.loads(open('gpurun_out/r02_bench_${cfg}_n2.json').read().strip().splitlines()[-1])
print('$cfg', d['n_gpus'], d['value'], 'e2e', d['e2e'] and d['e2e']['value'])"; done
