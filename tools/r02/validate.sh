#!/bin/bash
# Round-2 re-entry validation: GPU tests, smoke, default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/v_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/v_smoke.log)"
timeout 600 python bench.py > gpurun_out/v_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/v_bench.log
timeout 300 python tools/agg24_bench.py > gpurun_out/v_agg24.log 2>&1; echo "agg24 rc=$?"; cat gpurun_out/v_agg24.log | tail -4
GDX_P24_48=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/v_bench48off.log 2>&1; echo "p24_48 off: $(grep -o '"value": [0-9.]*' gpurun_out/v_bench48off.log | head -1)"
