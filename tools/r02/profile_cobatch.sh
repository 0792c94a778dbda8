#!/bin/bash
# ncu --set full of the cobatch kernels after the round-2 kernel choices (one GPU)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/prof3
mkdir -p $O
METRICS=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tma.sum
timeout 600 python tools/profile_target.py cobatch --epochs 1 > $O/plain_cobatch.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:aggregate|gemm_bf16x3' -s 0 -c 14 -o $O/full_cobatch \
    python tools/profile_target.py cobatch --epochs 1 > $O/ncu_cobatch.log 2>&1
echo "ncu rc=$?"
ncu -i $O/full_cobatch.ncu-rep --page raw --csv --metrics $METRICS > $O/full_cobatch.csv 2> $O/err.txt
rm -f $O/full_cobatch.ncu-rep
wc -l $O/full_cobatch.csv
