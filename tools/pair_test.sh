timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for pp in 1 0; do GDX_GEMM_PAIR=$pp timeout 300 python tools/gemm_bench.py > gpurun_out/gbp_$pp.log 2>&1; done
python3 - <<'PY'
import json
a=json.load(open("gpurun_out/gbp_1.log")); b=json.load(open("gpurun_out/gbp_0.log"))
for x,y in zip(a,b): print(f"{x['shape'][:40]:40s} pair {x['ms']:8.4f}  old {y['ms']:8.4f}")
PY
for pp in 1 0; do GDX_GEMM_PAIR=$pp timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bpr_$pp.log 2>&1; echo "reddit pair=$pp $(grep -o '"value": [0-9.]*' gpurun_out/bpr_$pp.log)"; GDX_GEMM_PAIR=$pp timeout 300 python bench.py --config products-gcn --no-cpu-baseline --no-e2e > gpurun_out/bpp_$pp.log 2>&1; echo "products pair=$pp $(grep -o '"value": [0-9.]*' gpurun_out/bpp_$pp.log)"; done
