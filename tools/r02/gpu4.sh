#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_parity_baseline.py -q -rA --durations=10 > gpurun_out/r02d_parity.log 2>&1
echo "rc=$?" >> gpurun_out/r02d_parity.log
( timeout 300 python tools/grad_precision.py
  timeout 300 python tools/grad_precision.py --n 3000 --deg 20 --dims 96,64,64,41 --lr 0.5 ) > gpurun_out/r02d_gradprec.jsonl 2>&1
tail -30 gpurun_out/r02d_parity.log; cat gpurun_out/r02d_gradprec.jsonl
