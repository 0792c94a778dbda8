#!/bin/bash
# packed-24 kernel: predicated remainder block vs the serial remainder loop (build/libgdx_base.so)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/tab; mkdir -p $O
timeout 900 python -m pytest -q -m gpu tests/test_gpu_kernels.py tests/test_native_trainer.py -x > $O/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest.log)"
for i in 1 2 3; do for v in base new; do
  if [ $v = base ]; then export GDX_LIB_PATH=$PWD/build/libgdx_base.so; else unset GDX_LIB_PATH; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-hbm-pass --no-e2e --no-cpu-baseline > $O/$v.json 2> $O/$v.err
  python -c "import json; d=json.loads(open('$O/$v.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', d['ms_per_step'], r['avg_launch_ms'], d['clocks']['sm_mhz'])" || tail -3 $O/$v.err
done; done
unset GDX_LIB_PATH
