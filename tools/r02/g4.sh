#!/bin/bash
# fused LOAD (TMA gather4 GEMM operands): kernel tests, cobatch tests, papers A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/g4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g4_tests.log
tail -3 gpurun_out/g4_tests.log
timeout 900 python -m pytest tests/test_cobatch.py -q -x > gpurun_out/g4_cobatch.log 2>&1; echo "rc=$?" >> gpurun_out/g4_cobatch.log
tail -3 gpurun_out/g4_cobatch.log
for v in 1 0 1; do
  GDX_FUSED_LOAD=$v timeout 2400 python bench.py --config papers-cobatch --steps 2 --warmup 3 > gpurun_out/g4_papers_$v.json 2> gpurun_out/g4_papers_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/g4_papers_$v.json').read().strip().splitlines()[-1]); print('papers fused_load=$v', d['ms_per_step'], d.get('parity',{}).get('abs_diff'), d['loss_after'], d['roofline']['frac'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/g4_papers_$v.err
done
