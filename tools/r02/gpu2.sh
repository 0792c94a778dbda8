#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
( for init in uniform he; do timeout 300 python tools/grad_precision.py --init $init; done
  timeout 300 python tools/grad_precision.py --n 3000 --deg 20 --dims 96,64,64,41 --lr 0.5
  timeout 300 python tools/grad_precision.py --kind gcn --n 2449029 --deg 25.26 --seed 13 --dims 100,64,64,47
) > gpurun_out/r02b_gradprec.jsonl 2>&1
cat gpurun_out/r02b_gradprec.jsonl
