R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python bench.py > gpurun_out/f2_r1.log 2>&1; echo "reddit N=1 $(grep -o '"value": [0-9.]*' gpurun_out/f2_r1.log | head -2 | tr '\n' ' ')"
for n in 2 4; do timeout 600 $R --nproc-per-node $n --master-port 2990$n bench.py --gpus $n > gpurun_out/f2_r$n.log 2>&1; echo "reddit N=$n $(grep -o '"value": [0-9.]*' gpurun_out/f2_r$n.log | head -2 | tr '\n' ' ')"; done
timeout 300 python bench.py --config products-gcn --no-cpu-baseline > gpurun_out/f2_p1.log 2>&1; echo "products N=1 $(grep -o '"value": [0-9.]*' gpurun_out/f2_p1.log | head -1)"
timeout 600 $R --nproc-per-node 4 --master-port 29911 bench.py --gpus 4 --config products-gcn --no-e2e > gpurun_out/f2_p4.log 2>&1; echo "products N=4 $(grep -o '"value": [0-9.]*' gpurun_out/f2_p4.log | head -1)"
timeout 900 $R --nproc-per-node 4 --master-port 29912 bench.py --config papers-cobatch --gpus 4 --steps 2 --warmup 1 > gpurun_out/f2_c4.log 2>&1; echo "papers N=4 $(grep -o '"value": [0-9.]*' gpurun_out/f2_c4.log | head -1)"
timeout 800 python bench.py --config papers-cobatch --steps 2 --warmup 1 > gpurun_out/f2_c1.log 2>&1; echo "papers N=1 $(grep -o '"value": [0-9.]*' gpurun_out/f2_c1.log | head -1)"
bash tools/profile_run.sh
