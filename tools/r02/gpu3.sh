#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
( timeout 300 python tools/gemm_precision.py
  timeout 300 python tools/gemm_precision.py --dist relu --n 64
  timeout 300 python tools/gemm_precision.py --k 3000 --splitks 1,3
) > gpurun_out/r02c_gemmprec.jsonl 2>&1
cat gpurun_out/r02c_gemmprec.jsonl
