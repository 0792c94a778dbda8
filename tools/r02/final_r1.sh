#!/bin/bash
# Final 1-GPU measurement of the round-2 tree: default bench line (with the gather-pattern
# probe), launch list of the bench command, ncu --set full of the Reddit epoch's kernels.
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/fin; mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/fin/bench.json').read().strip().splitlines()[-1])
r=d['roofline']; print('value', d['value'], 'e2e', d['e2e']['value'], 'parity', d['parity']['abs_diff'])
print('l2 frac', r['frac'], 'gather', r['gather_ceiling'])
PY
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-hbm-pass"
$CMD > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
METRICS=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__grid_size,smsp__inst_executed.sum
timeout 600 python tools/profile_target.py reddit --epochs 1 > $O/plain_reddit.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:aggregate|gemm_bf16x3|softmax' -s 0 -c 16 -o $O/full_reddit \
    python tools/profile_target.py reddit --epochs 1 > $O/ncu_reddit.log 2>&1
echo "reddit ncu rc=$?"
ncu -i $O/full_reddit.ncu-rep --page raw --csv --metrics $METRICS > $O/full_reddit.csv 2> $O/full_reddit.err
ncu -i $O/full_reddit.ncu-rep --page details --csv > $O/details_reddit.csv 2>> $O/full_reddit.err
gzip -f $O/details_reddit.csv; rm -f $O/full_reddit.ncu-rep
ls -la $O
