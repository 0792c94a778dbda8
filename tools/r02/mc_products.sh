#!/bin/bash
# products GCN at N=4: torch-orchestrated trainer with the SM push vs the NVSwitch multicast push
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/mc; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for i in 1 2; do for push in sm mc; do
  GDX_PUSH=$push timeout 600 $R --master-port 2960$i tools/trainer_compare.py --config products-gcn --steps 10 > $O/$push$i.log 2>&1
  echo "push=$push: $(grep '^{' $O/$push$i.log | tail -1)"
done; done
