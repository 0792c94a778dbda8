#!/bin/bash
# ncu --set full of the cooperative-batch kernels (row-group aggregation, sparse/full
# push not applicable on 1 GPU) on a papers-shape batch; one GPU.
export GDX_CONFIG=papers-cobatch GDX_N=30000000 GDX_R=64 GDX_NB=2
CMD="python tools/phase_breakdown.py"
mkdir -p gpurun_out
$CMD > gpurun_out/cob_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"aggregate_rows|gemm_bf16x3|gather_split_rows|grad_prepare" -s 30 -c 8 -o gpurun_out/prof_cobatch $CMD > gpurun_out/ncu_cobatch.log 2>&1
echo "cobatch profile rc=$?"
