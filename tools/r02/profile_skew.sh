#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/prof4; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 300 python tools/skew_bench.py > $O/skew.json 2>&1 && \
timeout 900 ncu --set full --clock-control none -k 'regex:aggregate|heavy' -s 14 -c 4 -o $O/skew python tools/skew_bench.py > $O/ncu.log 2>&1
ncu -i $O/skew.ncu-rep --page raw --csv --metrics $M > $O/skew.csv 2>/dev/null; rm -f $O/skew.ncu-rep
cat $O/skew.json; cut -c1-400 $O/skew.csv | head -8
