#!/bin/bash
# Launch list only (gpu__time_duration per kernel) of a short bench run, on one GPU.
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --eager"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
