#!/bin/bash
# ncu --set full of the output launch (GW) on the N=2^18 product-compress c3-shaped tree, then the
# SASS context of its hottest stall sites (which barrier / load a stall belongs to) on the box.
set -u
mkdir -p gpurun_out /tmp/prof
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:grouped_gemm_f64" \
    --launch-skip 18 --launch-count 1 -o /tmp/prof/gwo python tools/profile_run.py --n 262144 --tree compress \
    --evals 1 > gpurun_out/gwo_ncu.log 2>&1
echo "capture rc=$?"
ncu -i /tmp/prof/gwo.ncu-rep --page source --csv --print-source sass > /tmp/prof/gwo_src.csv 2>&1
python tools/ncu_hot_context.py /tmp/prof/gwo_src.csv 8 10 > gpurun_out/gwo_hot_context.txt 2>&1
python tools/ncu_source_top.py /tmp/prof/gwo_src.csv 40 > gpurun_out/gwo_source_top.txt 2>&1
python tools/ncu_summary.py /tmp/prof/gwo.ncu-rep > gpurun_out/gwo_summary.txt 2>&1
ncu -i /tmp/prof/gwo.ncu-rep --page details --csv > gpurun_out/gwo_details.csv 2>&1
echo done
