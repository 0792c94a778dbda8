#!/bin/bash
# mask-TMA dH GEMM A/B + the GEMM tests + products / papers benches
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" > gpurun_out/tma_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tma_tests.log
tail -3 gpurun_out/tma_tests.log
for v in 1 0; do
  GDX_MASK_TMA=$v GEMM_ONLY=fused timeout 600 python tools/gemm_bench.py > gpurun_out/tma2_gemm_$v.json 2> gpurun_out/tma2_gemm_$v.err
done
python - <<'PY'
import json
a={d['shape']:d for d in json.load(open('gpurun_out/tma2_gemm_1.json'))}
b={d['shape']:d for d in json.load(open('gpurun_out/tma2_gemm_0.json'))}
for k in a: print(f"{k:48s} masktma {a[k]['ms']:.4f} ({a[k]['GBps']:.0f} GB/s)  old {b[k]['ms']:.4f} ({b[k]['GBps']:.0f})")
PY
for v in 1 0; do
  GDX_MASK_TMA=$v timeout 600 python bench.py --config products-gcn --steps 10 --warmup 3 --no-hbm-pass > gpurun_out/tma2_products_$v.json 2> gpurun_out/tma2_products_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/tma2_products_$v.json').read().strip().splitlines()[-1]); print('products masktma=$v', d['ms_per_step'], d['parity']['abs_diff'], d['roofline']['tensor']['share_of_step'])"
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-hbm-pass > gpurun_out/tma2_reddit.json 2> gpurun_out/tma2_reddit.err
python -c "import json; d=json.loads(open('gpurun_out/tma2_reddit.json').read().strip().splitlines()[-1]); print('reddit', d['ms_per_step'], d['parity']['abs_diff'], d['e2e']['value'])"
timeout 2400 python bench.py --config papers-cobatch --steps 2 --warmup 3 > gpurun_out/tma2_papers.json 2> gpurun_out/tma2_papers.err
python -c "import json; d=json.loads(open('gpurun_out/tma2_papers.json').read().strip().splitlines()[-1]); print('papers', d['value'], d['ms_per_step'], d.get('parity'), d['roofline']['frac'])"
