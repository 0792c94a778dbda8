#!/bin/bash
# packed-24 gather: the remote-source pass walks both sides of the skip hole as one edge
# stream (new) vs two segments (build/libgdx_base.so); correctness first
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/hab; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest -q -m gpu tests/test_gpu_kernels.py tests/test_balanced.py tests/test_native_trainer.py tests/test_multi_gpu.py -x > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
for n in 1 4 2; do for i in 1 2; do for v in base new; do
  if [ $v = base ]; then export GDX_LIB_PATH=$PWD/build/libgdx_base.so; else unset GDX_LIB_PATH; fi
  timeout 600 $R --nproc-per-node $n --master-port 297$n$i bench.py --gpus $n --steps 20 --warmup 5 --no-hbm-pass --no-e2e --no-cpu-baseline > $O/$v$n.json 2> $O/$v$n.err
  python -c "import json; d=json.loads(open('$O/$v$n.json').read().strip().splitlines()[-1]); r=d['roofline']; print('N=$n $v', d['ms_per_step'], r['avg_launch_ms'])" || tail -3 $O/$v$n.err
done; done; done
unset GDX_LIB_PATH
