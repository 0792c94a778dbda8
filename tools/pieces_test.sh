R="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for n in 2 4; do timeout 300 $R $n --master-addr 127.0.0.1 --master-port 2951$n tools/dist_check.py > gpurun_out/dp$n.log 2>&1; echo "dist N=$n $(grep -o '"ok": [a-z]*' gpurun_out/dp$n.log | head -1)"; grep -iE "Error|Traceback" gpurun_out/dp$n.log | head -3; done
for n in 2 4; do for pc in 1 0; do
  if [ $pc = 1 ]; then unset GDX_AGG_PIECES; else export GDX_AGG_PIECES=1; fi
  timeout 300 $R $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bp_${n}_$pc.log 2>&1; echo "reddit N=$n pieces=$pc $(grep -o '"value": [0-9.]*' gpurun_out/bp_${n}_$pc.log)"
done; done
unset GDX_AGG_PIECES
timeout 300 $R 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --config products-gcn --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bp_prod4.log 2>&1; echo "products N=4 pieces $(grep -o '"value": [0-9.]*' gpurun_out/bp_prod4.log)"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
