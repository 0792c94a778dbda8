#!/bin/bash
# Re-entry 3 validation: whole -m gpu suite, smoke, default bench line, launch list.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/e3_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/e3_pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e3_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/e3_smoke.log)"
timeout 600 python bench.py > gpurun_out/e3_bench.json 2> gpurun_out/e3_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/e3_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/e3_ref.json 2> gpurun_out/e3_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/e3_ref.json
