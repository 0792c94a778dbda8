R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29511 tools/dist_check.py > gpurun_out/d4s.log 2>&1; echo "dist $(grep -o '"ok": [a-z]*' gpurun_out/d4s.log | head -1)"; grep -iE "error|Traceback" gpurun_out/d4s.log | head -3
for sp in 1 0; do GDX_SPARSE_PUSH=$sp GDX_N=30000000 GDX_R=64 GDX_CONFIG=papers-cobatch GDX_NB=4 timeout 600 $R --master-port 29521 tools/phase_breakdown.py > gpurun_out/cob_sp$sp.log 2>&1; grep "^{" gpurun_out/cob_sp$sp.log; done
timeout 900 $R --master-port 29513 bench.py --config papers-cobatch --gpus 4 --steps 2 --warmup 1 > gpurun_out/bench_papers4s.log 2>&1; grep -o '"value": [0-9.]*, "unit": "ms", "n_gpus": [0-9]' gpurun_out/bench_papers4s.log
