#!/bin/bash
# alternating A/B of an env knob on a bench config: ab.sh CONFIG VAR VALUE_A VALUE_B [ROUNDS]
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CFG=$1; VAR=$2; A=$3; B=$4; R=${5:-3}
for i in $(seq 1 $R); do
  for v in $A $B; do
    env $VAR=$v timeout 600 python bench.py --config $CFG --steps 20 --warmup 5 --no-hbm-pass > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$CFG $VAR=$v', d['ms_per_step'], d['clocks']['sm_mhz'], round(d['roofline']['tensor']['share_of_step']*d['ms_per_step'],3), d['parity']['ok'])"
  done
done
