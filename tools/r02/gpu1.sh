#!/bin/bash
# round-2 GPU session 1: gpu tests (incl. BASELINE-size parity), headline bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/r02a_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
echo "bench rc=$?" >> gpurun_out/r02a_bench.err
tail -3 gpurun_out/r02a_pytest_gpu.log
cat gpurun_out/r02a_bench.json | head -c 3000
