#!/bin/bash
# Round-2 profiling (ONE GPU): launch list of the bench command, ncu --set full of the
# aggregation / GEMM kernels per workload.  Each ncu run only after its command exits 0.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/prof2
O=gpurun_out/prof2
METRICS=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__grid_size,smsp__inst_executed.sum,sm__inst_executed_pipe_tma.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
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
  # the reports are ~60 MB each: keep the metrics as CSV, drop the report (gpurun copies <= 64 MiB back)
  ncu -i $O/full_$t.ncu-rep --page raw --csv --metrics $METRICS > $O/full_$t.csv 2> $O/full_$t.err
  ncu -i $O/full_$t.ncu-rep --page details --csv > $O/details_$t.csv 2>> $O/full_$t.err
  gzip -f $O/details_$t.csv
  rm -f $O/full_$t.ncu-rep
done
ls -la $O
