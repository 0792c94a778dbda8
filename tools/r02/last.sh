#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/last; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $O/smoke.log)"
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['parity']['abs_diff'], d['roofline']['frac'], d['roofline']['gather_ceiling']['frac'], d['clocks'])"
