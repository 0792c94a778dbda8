#!/bin/bash
# predicated-tail A/B for the low-degree row-group aggregation: build/libgdx_base.so = previous build
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for deg in 3 6 12; do  # variants 1,2
  for lib in build/libgdx_base.so paper_2311_06837_b200/libgdx.so; do
    GDX_LIB_PATH=$PWD/$lib timeout 600 python tools/agg_bench.py --n 6000000 --degree $deg --widths 64 --variants 1,2 --no-probe > gpurun_out/tail.json 2>gpurun_out/tail.err
    python -c "
import json
for r in json.loads(open('gpurun_out/tail.json').read().strip().splitlines()[-1]): print('$lib'.split('/')[-1], 'deg', r['deg'], 'variant', r['variant'], r['ms'], r['alg_GBps'])
"
  done
done
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_balanced.py -q -x > gpurun_out/tail_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tail_tests.log; tail -2 gpurun_out/tail_tests.log
for lib in build/libgdx_base.so paper_2311_06837_b200/libgdx.so; do
  GDX_LIB_PATH=$PWD/$lib timeout 2400 python bench.py --config papers-cobatch --steps 2 --warmup 3 > gpurun_out/tail_papers.json 2> gpurun_out/tail_papers.err
  python -c "import json; d=json.loads(open('gpurun_out/tail_papers.json').read().strip().splitlines()[-1]); print('$lib papers', d['ms_per_step'], d.get('parity',{}).get('abs_diff'), d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
