#!/bin/bash
# Final tree: whole -m gpu suite, smoke, ncu launch list of the default bench command
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/vf; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --durations=8 > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)"
