#!/bin/bash
# Round-2 profiling (ONE GPU): launch list of the bench command, ncu --set full of the
# aggregation / GEMM kernels per workload.  Each ncu run only after its command exits 0.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/prof2
O=gpurun_out/prof2
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-hbm-pass"
$CMD > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
for t in reddit products hbm cobatch; do
  timeout 600 python tools/profile_target.py $t --epochs 1 > $O/plain_$t.log 2>&1 || { echo "$t plain failed"; continue; }
  case $t in
    reddit)   K='regex:aggregate|gemm_bf16x3'; S=0; N=14 ;;
    products) K='regex:aggregate|gemm_bf16x3'; S=0; N=14 ;;
    hbm)      K='regex:aggregate'; S=3; N=1 ;;
    cobatch)  K='regex:aggregate|gemm_bf16x3'; S=0; N=14 ;;
  esac
  timeout 1500 ncu --set full --clock-control none --import-source on -k "$K" -s $S -c $N -o $O/full_$t \
    python tools/profile_target.py $t --epochs 1 > $O/ncu_$t.log 2>&1
  echo "$t ncu rc=$?"
done
ls -la $O
