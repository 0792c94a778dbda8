#!/bin/bash
# packed-24 trainer rows: GPU tests + Reddit / gcn56 A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "packed24 or gemm" > gpurun_out/p24_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p24_tests.log
tail -3 gpurun_out/p24_tests.log
timeout 900 python -m pytest tests/test_native_trainer.py -q -x > gpurun_out/p24_trainer.log 2>&1; echo "rc=$?" >> gpurun_out/p24_trainer.log
tail -3 gpurun_out/p24_trainer.log
for i in 1; do for v in 1 0; do
  GDX_PACKED24=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-hbm-pass > gpurun_out/p24_reddit_$v.json 2> gpurun_out/p24_reddit_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/p24_reddit_$v.json').read().strip().splitlines()[-1]); print('reddit p24=$v', d['ms_per_step'], d['parity']['abs_diff'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])" || tail -5 gpurun_out/p24_reddit_$v.err
done; done
for v in 1 0; do
  GDX_PACKED24=$v timeout 900 python bench.py --config reddit-gcn56-eas --steps 5 --warmup 3 --no-hbm-pass > gpurun_out/p24_gcn56_$v.json 2> gpurun_out/p24_gcn56_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/p24_gcn56_$v.json').read().strip().splitlines()[-1]); print('gcn56 p24=$v', d['ms_per_step'], d.get('parity',{}).get('abs_diff'), d['loss_after'])" || tail -5 gpurun_out/p24_gcn56_$v.err
done
