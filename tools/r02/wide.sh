#!/bin/bash
# 48-wide packed-24 wide-gather variant: kernel A/B, GPU kernel tests, bench A/B
mkdir -p gpurun_out
timeout 300 python tools/agg24_bench.py > gpurun_out/w_agg24.log 2>&1; echo "agg24 rc=$?"; grep '"width": 48' gpurun_out/w_agg24.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_native_trainer.py -q -x -m gpu > gpurun_out/w_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/w_pytest.log)"
for v in 1 0; do GDX_P24_WIDE=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/w_bench$v.log 2>&1; echo "wide=$v: $(grep -o '"value": [0-9.]*' gpurun_out/w_bench$v.log | head -1) $(grep -o '"abs_diff": [0-9.e-]*' gpurun_out/w_bench$v.log)"; done
