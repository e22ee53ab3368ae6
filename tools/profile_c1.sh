#!/bin/bash
# c1 (latency-bound): ncu --set full of every grouped-GEMM launch of one evaluation on the
# product-compress c1 tree, summarised per launch (duration, cycles, stalls) on the box.
set -u
mkdir -p gpurun_out /tmp/prof
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm_f64" \
    --launch-skip 13 --launch-count 13 -o /tmp/prof/c1 python tools/latency_probe.py c1 --reps 2 \
    > gpurun_out/ncu_c1.log 2>&1
echo "capture rc=$?"
ncu -i /tmp/prof/c1.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.avg,smsp__warps_issue_stalled_barrier_per_warp_active.pct,smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct,smsp__warps_issue_stalled_membar_per_warp_active.pct,smsp__warps_issue_stalled_wait_per_warp_active.pct,smsp__warps_issue_stalled_sleeping_per_warp_active.pct,smsp__inst_executed.sum,dram__bytes_read.sum,launch__grid_size,smsp__cycles_active.avg,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__warps_issue_stalled_math_pipe_throttle_per_warp_active.pct,smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__warps_issue_stalled_mio_throttle_per_warp_active.pct \
    > gpurun_out/ncu_c1_raw.csv 2>&1
for i in 0 5 12; do
  ncu -i /tmp/prof/c1.ncu-rep --launch-skip $i --launch-count 1 --page source --csv --print-source sass \
      > /tmp/prof/src_$i.csv 2>&1
  python tools/ncu_source_top.py /tmp/prof/src_$i.csv 40 > gpurun_out/ncu_c1_src_$i.txt 2>&1
done
ncu -i /tmp/prof/c1.ncu-rep --page details --csv > gpurun_out/ncu_c1_details.csv 2>&1
echo done
