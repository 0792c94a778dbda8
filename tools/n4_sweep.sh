#!/bin/bash
# Reddit SAGE at N=4 under the exchange knobs (DESIGN §4 alternatives); one line each.
mkdir -p gpurun_out
run() {
  env "$@" timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --no-cpu-baseline --no-e2e 2>&1 \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], d['value'])" "$*"
}
run X=0
run GDX_PUSH_CTAS=16
run GDX_PUSH_CTAS=64
run GDX_PUSH_CTAS=148
run GDX_P2P_SPLIT=0
run GDX_EXCHANGE=nccl
run X=0
