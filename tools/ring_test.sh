R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29511 tools/dist_check.py > gpurun_out/d4r.log 2>&1; echo "dist $(grep -o '"ok": [a-z]*' gpurun_out/d4r.log | head -1)"; grep -iE "error|Traceback" gpurun_out/d4r.log | head -3
for ring in 1 0; do
  GDX_P2P_RING=$ring timeout 300 $R --master-port 29512 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/rr_$ring.log 2>&1; echo "reddit ring=$ring $(grep -o '"value": [0-9.]*' gpurun_out/rr_$ring.log)"
  GDX_P2P_RING=$ring timeout 300 $R --master-port 29513 bench.py --gpus 4 --config products-gcn --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/rp_$ring.log 2>&1; echo "products ring=$ring $(grep -o '"value": [0-9.]*' gpurun_out/rp_$ring.log)"
done
GDX_N=30000000 GDX_R=64 GDX_CONFIG=papers-cobatch GDX_NB=4 timeout 600 $R --master-port 29521 tools/phase_breakdown.py > gpurun_out/cob_ring.log 2>&1; grep "^{" gpurun_out/cob_ring.log
