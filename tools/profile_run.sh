#!/bin/bash
# Profiling recipe (run under gpurun on ONE GPU): plain run, launch list, ncu --set full
# of the aggregation and GEMM kernels.  Outputs land in gpurun_out/.
set -u
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"aggregate_vec4|aggregate_rows|gemm_bf16x3" -s 40 -c 6 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "profile done rc=$?"
