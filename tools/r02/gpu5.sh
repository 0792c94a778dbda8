#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
./build/ref_suite_b200 > gpurun_out/r02e_refsuite.txt 2>&1; echo "rc=$?" >> gpurun_out/r02e_refsuite.txt
timeout 900 python -m pytest tests/test_cobatch_planner.py tests/test_cobatch.py tests/test_golden.py tests/test_reference_suite.py -q -rf > gpurun_out/r02e_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r02e_pytest.log
tail -25 gpurun_out/r02e_pytest.log; grep -E "FAIL|ref-suite" gpurun_out/r02e_refsuite.txt | head -20
