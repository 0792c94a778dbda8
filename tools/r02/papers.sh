#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${1:-1}
if [ $N = 1 ]; then
  timeout 2400 python bench.py --config papers-cobatch --steps 2 --warmup 3 > gpurun_out/r02_bench_papers_n1.json 2> gpurun_out/r02_bench_papers_n1.err
else
  timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29581 \
    bench.py --gpus $N --config papers-cobatch --steps 2 --warmup 3 > gpurun_out/r02_bench_papers_n$N.json 2> gpurun_out/r02_bench_papers_n$N.err
fi
echo "rc=$?" >> gpurun_out/r02_bench_papers_n$N.err
tail -3 gpurun_out/r02_bench_papers_n$N.err
python -c "
import json
d=json.loads(open('gpurun_out/r02_bench_papers_n$N.json').read().strip().splitlines()[-1])
print(d['value'], d['cuda_graph'], d['loss_after'], d.get('parity'), d['roofline']['frac'], d['setup_s'])
"
