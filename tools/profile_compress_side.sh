#!/bin/bash
# ncu DRAM bytes / duration of the §8(f) kernels: batched skeletonisation (444 c3-shaped nodes =
# one full wave at 3 per SM) and the ANN leaf pass (N=2^18, m=512, kappa=32).
set -u
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k regex:skeletonize_kernel --csv --log-file gpurun_out/ncu_skel.csv \
    python tools/bench_skel.py --nodes 444 --cpu-nodes 2 > gpurun_out/ncu_skel.log 2>&1; echo "skel rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k regex:ann_leaf_kernel --csv --log-file gpurun_out/ncu_ann.csv \
    python tools/bench_ann.py > gpurun_out/ncu_ann.log 2>&1; echo "ann rc=$?"
