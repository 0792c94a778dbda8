#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_native_trainer.py -q -rf -x > gpurun_out/r02f_native.log 2>&1
echo "rc=$?" >> gpurun_out/r02f_native.log
tail -40 gpurun_out/r02f_native.log
