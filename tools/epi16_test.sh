timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python tools/gemm_bench.py > gpurun_out/gb16.log 2>&1
python3 -c "
import json
for r in json.load(open('gpurun_out/gb16.log')): print(f\"{r['shape'][:40]:40s} {r['ms']:8.4f}\")"
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b16r.log 2>&1; echo "reddit $(grep -o '"value": [0-9.]*' gpurun_out/b16r.log)"
timeout 300 python bench.py --config products-gcn --no-cpu-baseline --no-e2e > gpurun_out/b16p.log 2>&1; echo "products $(grep -o '"value": [0-9.]*' gpurun_out/b16p.log)"
