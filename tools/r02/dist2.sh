#!/bin/bash
# multi-GPU correctness: every exchange mode (tools/dist_check.py) at N = $1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${1:-2}
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29555 tools/dist_check.py --out gpurun_out/r02_dist_check_n$N.json > gpurun_out/r02_dist_n$N.log 2>&1
echo "rc=$?" >> gpurun_out/r02_dist_n$N.log
tail -5 gpurun_out/r02_dist_n$N.log | cut -c1-3000
python - <<PY
import json
d=json.load(open("gpurun_out/r02_dist_check_n$N.json"))
print("world", d["world"], "ok", d["ok"])
for m, r in d["modes"].items():
    print(m, r.get("ok"), r.get("skipped",""), r.get("error",""), r.get("seconds"),
          [c.get("max_abs_loss_diff") for c in r.get("cases", [])])
PY
