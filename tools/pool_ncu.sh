#!/usr/bin/env bash
# ncu --set full of the c3 pool1 max-pool kernels (smem vs streaming, forward with tanh and
# backward), summarised on the box: bash tools/pool_ncu.sh <outdir>
OUT=${1:-gpurun_out/pool_ncu}; mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard,smsp__average_warp_latency_issue_stalled_short_scoreboard,smsp__average_warp_latency_issue_stalled_barrier,smsp__average_warp_latency_issue_stalled_mio_throttle,smsp__average_warp_latency_issue_stalled_lg_throttle,smsp__average_warp_latency_issue_stalled_wait,smsp__average_warp_latency_issue_stalled_math_pipe_throttle,smsp__average_warp_latency_issue_stalled_no_instruction,smsp__average_warp_latency_issue_stalled_dispatch_stall,smsp__average_warp_latency_issue_stalled_membar,launch__registers_per_thread,launch__occupancy_limit_shared_mem,sm__maximum_warps_per_active_cycle_pct
for K in maxpool_fwd_smem maxpool_fwd_stream maxpool_bwd_smem maxpool_bwd_stream; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 \
     -o $OUT/$K -f python tools/pool_ab.py 1 > $OUT/$K.log 2>&1
  ncu -i $OUT/$K.ncu-rep --page raw --csv --metrics $M > $OUT/$K.csv 2>&1
  ncu -i $OUT/$K.ncu-rep --page source --csv > $OUT/$K.src.csv 2>&1
done
ls -la $OUT
