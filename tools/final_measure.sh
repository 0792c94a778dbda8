R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 2 4; do timeout 600 $R --nproc-per-node $n --master-port 2970$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/final_r$n.log 2>&1; echo "reddit N=$n $(grep -o '"value": [0-9.]*' gpurun_out/final_r$n.log | head -2 | tr '\n' ' ')"; done
timeout 600 $R --nproc-per-node 4 --master-port 29710 bench.py --gpus 4 --config products-gcn --no-e2e > gpurun_out/final_p4.log 2>&1; echo "products N=4 $(grep -o '"value": [0-9.]*' gpurun_out/final_p4.log | head -1)"
timeout 600 python bench.py > gpurun_out/final_r1.log 2>&1; echo "reddit N=1 $(grep -o '"value": [0-9.]*' gpurun_out/final_r1.log | head -2 | tr '\n' ' ')"
bash tools/profile_run.sh
