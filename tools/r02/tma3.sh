#!/bin/bash
# staged (TMA-store) epilogue threshold A/B on the short Reddit GEMMs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in 0 1048576; do
  GDX_STAGE_MIN_ROWS=$v timeout 600 python tools/gemm_bench.py > gpurun_out/tma3_gemm_$v.json 2> gpurun_out/tma3_gemm_$v.err
done
python - <<'PY'
import json
a={d['shape']:d for d in json.load(open('gpurun_out/tma3_gemm_0.json'))}
b={d['shape']:d for d in json.load(open('gpurun_out/tma3_gemm_1048576.json'))}
for k in a: print(f"{k:48s} staged-all {a[k]['ms']:.4f} ({a[k]['GBps']:.0f} GB/s)  >=1M {b[k]['ms']:.4f} ({b[k]['GBps']:.0f})")
PY
for v in 0 1048576; do
GDX_STAGE_MIN_ROWS=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-hbm-pass > gpurun_out/tma3_reddit_$v.json 2> gpurun_out/tma3_reddit_$v.err
python -c "import json; d=json.loads(open('gpurun_out/tma3_reddit_$v.json').read().strip().splitlines()[-1]); print('reddit $v', d['ms_per_step'], d['parity']['abs_diff'], d['roofline']['tensor']['share_of_step'])"
done
GDX_STAGE_MIN_ROWS=0 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_native_trainer.py -q -x > gpurun_out/tma3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tma3_tests.log
tail -2 gpurun_out/tma3_tests.log
