#!/bin/bash
# TMA-store epilogue A/B: GEMM parity tests, gemm_bench with and without, products + cobatch bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/tma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tma_tests.log
tail -3 gpurun_out/tma_tests.log
for v in 1 0; do
  GDX_GEMM_TMA_STORE=$v timeout 600 python tools/gemm_bench.py > gpurun_out/tma_gemm_$v.json 2> gpurun_out/tma_gemm_$v.err
done
python - <<'PY'
import json
a={d['shape']:d for d in json.load(open('gpurun_out/tma_gemm_1.json'))}
b={d['shape']:d for d in json.load(open('gpurun_out/tma_gemm_0.json'))}
for k in a: print(f"{k:48s} tma {a[k]['ms']:.4f} ({a[k]['GBps']:.0f} GB/s)  old {b[k]['ms']:.4f} ({b[k]['GBps']:.0f})")
PY
for v in 1 0; do
  GDX_GEMM_TMA_STORE=$v timeout 600 python bench.py --config products-gcn --steps 10 --warmup 3 --no-hbm-pass > gpurun_out/tma_products_$v.json 2> gpurun_out/tma_products_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/tma_products_$v.json').read().strip().splitlines()[-1]); print('products tma=$v', d['ms_per_step'], d['parity'])"
done
